# generic A/B of one variant against the default build: bash tools/ab_v.sh build/variants/x.so
mkdir -p gpurun_out
B=paper_1403_6870_b200/libzigfast_b200.so
V=$1
out=gpurun_out/ab_v.txt
: > $out
for n in 32 28; do
  reps=$(( n >= 32 ? 3 : 20 ))
  python tools/ab.py --n $n --reps $reps --rounds 4 --cool 1 $B $V 2>&1 | grep '@1965\|differ' >> $out
done
python tools/ab.py --n 32 --reps 20 --rounds 2 --cool 3 $B $V 2>&1 | grep 'n=2' >> $out
python tools/ab.py --n 30 --sustain 2.0 --rounds 2 --cool 3 --dists normal $B $V >> $out 2>&1
