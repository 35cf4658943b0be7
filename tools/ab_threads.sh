mkdir -p gpurun_out
B=paper_1403_6870_b200/libzigfast_b200.so
V=build/variants
: > gpurun_out/abwv_32.txt
for w in 6 12 24 48; do
  echo "== waves $w" >> gpurun_out/abwv_32.txt
  ZF_GRID_WAVES=$w python tools/ab.py --n 32 --reps 3 --rounds 3 --cool 1 $B $V/w16.so 2>&1 | grep '@1965' >> gpurun_out/abwv_32.txt
done
