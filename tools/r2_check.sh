# round-2 driver-equivalent check: GPU tests, smoke, bench (both arms)
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/r2_gputests.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_gputests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/r2_smoke.txt
timeout 900 python3 bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2_bench3.json 2> gpurun_out/r2_bench3.err; echo "bench rc=$?" >> gpurun_out/r2_bench3.err
timeout 900 python3 bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2_bench3_ref.json 2> gpurun_out/r2_bench3_ref.err
