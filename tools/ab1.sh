timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/r2_gputests.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_gputests.txt
timeout 600 python tools/bench_configs.py c5 > gpurun_out/r02_c5.jsonl 2>&1
