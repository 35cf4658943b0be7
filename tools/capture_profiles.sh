# ncu evidence for profiles/ (one GPU; run only after the same commands exit 0 without ncu):
#   gpurun -- bash tools/capture_profiles.sh
# then here: python tools/launch_summary.py gpurun_out/launches_bench.csv
#            python tools/ncu_summary.py gpurun_out/fill_*_f64_2p28.ncu-rep
set -e
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_bench.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_bench.log 2>&1
for d in normal exp; do
  ncu --set full --import-source on --clock-control none -k regex:fill_ctr_kernel -c 1 \
      -o gpurun_out/fill_${d}_f64_2p28 -f python tools/prof_fill.py $d 28 1 > gpurun_out/ncu_$d.log 2>&1
done
