timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/r2_gputests.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_gputests.txt
timeout 300 python tools/bench_configs.py c4 > gpurun_out/r2_c4.json 2>&1
