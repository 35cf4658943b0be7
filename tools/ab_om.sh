mkdir -p gpurun_out
: > gpurun_out/ab_om.txt
timeout 900 python -m pytest tests/test_gpu_oracle_mode.py tests/test_gpu_traditional.py tests/test_gpu_acceptance.py tests/test_gpu_checked.py tests/test_gpu_output.py -q -x > gpurun_out/om_tests.txt 2>&1
for n in 26 22 20; do
  python tools/ab_oracle.py --n $n --rounds 5 --reps 10 build/variants/om_prev.so paper_1403_6870_b200/libzigfast_b200.so >> gpurun_out/ab_om.txt 2>&1
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/om_launches26.csv python tools/oracle_prof.py 26 1 exp > /dev/null 2>&1
