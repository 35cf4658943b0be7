# round-2 check: GPU tests, then the default bench, then the reference arm
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/r2_gputests.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_gputests.txt
timeout 600 python bench.py > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err; echo "bench rc=$?" >> gpurun_out/r2_bench.err
python tools/prof_fill.py normal 32 1 > gpurun_out/r2_pf.txt 2>&1 && \
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:fill_ctr -c 1 --csv python tools/prof_fill.py normal 32 1 > gpurun_out/r2_ncu_traffic_2p32.csv 2>&1
