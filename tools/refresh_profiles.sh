# Re-measure every bench line of the round on one B200 (no profiler attached);
# outputs land in gpurun_out/ and are copied to profiles/ by hand.
set -e
mkdir -p gpurun_out
python bench.py > gpurun_out/r01_bench_line.json
python bench.py --impl reference > gpurun_out/r01_bench_reference_line.json
python bench.py --n 4294967296 --steps 10 --no-e2e --no-cpu-baseline > gpurun_out/r01_c3_bench_2p32.json
python tools/c5_multi.py 36 > gpurun_out/r01_c5_full_2p36.json
python tools/bench_configs.py c1 c1big c4 c5 f32 agg trad fmt > gpurun_out/r01_configs.jsonl
python tools/host_fill_probe.py > gpurun_out/r01_host_fill.txt
