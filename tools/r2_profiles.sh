# round-2 evidence: ncu captures of the final fill kernels, the bench launch list,
# DRAM traffic of one config-3 launch, and the generator battery at 2^38 words
set -x
python tools/prof_fill.py normal 28 2 > gpurun_out/p_plain1.txt 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:fill_ctr -s 2 -c 1 -o gpurun_out/r02_fill_normal_f64_2p28 python tools/prof_fill.py normal 28 2 > gpurun_out/p_ncu1.log 2>&1
python tools/prof_fill.py exp 28 2 > gpurun_out/p_plain2.txt 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:fill_ctr -s 2 -c 1 -o gpurun_out/r02_fill_exp_f64_2p28 python tools/prof_fill.py exp 28 2 > gpurun_out/p_ncu2.log 2>&1
python tools/prof_fill.py normal 32 1 > gpurun_out/p_plain3.txt 2>&1 && \
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:fill_ctr -c 1 --csv python tools/prof_fill.py normal 32 1 > gpurun_out/r02_ncu_traffic_2p32.csv 2>&1
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --c5-total 1073741824 > gpurun_out/p_plain4.txt 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches_bench.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --c5-total 1073741824 > gpurun_out/p_ncu4.log 2>&1
timeout 1800 python tools/battery.py --log2n 38 --seeds 7,1234,99,2024 --aval-log2m 24 --out gpurun_out/r02_battery.json > gpurun_out/r02_battery.txt 2>&1
