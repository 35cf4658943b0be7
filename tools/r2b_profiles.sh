# round-2 evidence after the grid-sizing change: ncu --set full of the headline
# kernels at the bench's own size (2^32), DRAM traffic of one config-3 launch,
# and the bench launch list (each command first runs once without ncu)
set -x
mkdir -p gpurun_out
for d in normal exp; do
  python tools/prof_fill.py $d 32 1 > gpurun_out/p_plain_$d.txt 2>&1 && \
  ncu --set full --import-source on --clock-control none -k regex:fill_ctr -s 1 -c 1 -o gpurun_out/r02b_fill_${d}_f64_2p32 -f python tools/prof_fill.py $d 32 1 > gpurun_out/p_ncu_$d.log 2>&1
done
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:fill_ctr -c 1 --csv python tools/prof_fill.py normal 32 1 > gpurun_out/r02b_ncu_traffic_2p32.csv 2>&1
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --c5-total 1073741824 > gpurun_out/p_plain_bench.txt 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02b_launches_bench.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --c5-total 1073741824 > gpurun_out/p_ncu_bench.log 2>&1
