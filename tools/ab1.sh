timeout 900 python -m pytest tests/test_gpu_oracle_mode.py tests/test_gpu_traditional.py -q -x > gpurun_out/om_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/om_tests.txt
python tools/oracle_prof.py 20 20 exp > gpurun_out/c1_plain.txt 2>&1
python tools/oracle_prof.py 20 20 normal >> gpurun_out/c1_plain.txt 2>&1
timeout 300 python tools/bench_configs.py c1 >> gpurun_out/c1_plain.txt 2>&1
