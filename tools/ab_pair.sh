# paired-tile build (default) vs the single-tile build saved as build/variants/single.so
mkdir -p gpurun_out
B=paper_1403_6870_b200/libzigfast_b200.so
S=build/variants/single.so
out=gpurun_out/ab_pair.txt
: > $out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pair_tests.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pair_tests.txt
for n in 32 28; do
  reps=$(( n >= 32 ? 3 : 20 ))
  python tools/ab.py --n $n --reps $reps --rounds 4 --cool 1 $S $B 2>&1 | grep '@1965\|differ' >> $out
done
python tools/ab.py --n 28 --dtype f32 --reps 20 --rounds 4 --cool 1 $S $B 2>&1 | grep '@1965\|differ' >> $out
python tools/bench_configs.py c4 c5 agg trad > gpurun_out/pair_configs.jsonl 2>&1
