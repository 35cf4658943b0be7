# final-state evidence (round 2, session d): ncu --set full of the headline kernel at
# the bench's own size, its DRAM traffic, and the bench launch list (every
# command first runs once without ncu)
set -x
mkdir -p gpurun_out
python tools/prof_fill.py normal 32 1 > gpurun_out/p_plain_normal.txt 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:fill_ctr -s 1 -c 1 -o gpurun_out/r02d_fill_normal_f64_2p32 -f python tools/prof_fill.py normal 32 1 > gpurun_out/p_ncu_normal.log 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:fill_ctr -c 1 --csv python tools/prof_fill.py normal 32 1 > gpurun_out/r02d_ncu_traffic_2p32.csv 2>&1
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --c5-total 1073741824 > gpurun_out/p_plain_bench.txt 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02d_launches_bench.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --c5-total 1073741824 > gpurun_out/p_ncu_bench.log 2>&1
python tools/launch_summary.py gpurun_out/r02d_launches_bench.csv > gpurun_out/r02d_launches_bench.summary.txt
