# cool A/B, sustained energy and bench-length rate of library builds
mkdir -p gpurun_out
out=gpurun_out/power_ab.txt
: > $out
python tools/ab.py --n 32 --reps 3 --rounds 3 --cool 1 "$@" 2>&1 | grep '@1965\|differ' >> $out
python tools/ab.py --n 30 --sustain 2.0 --rounds 2 --cool 3 --dists normal "$@" >> $out 2>&1
python tools/ab.py --n 32 --reps 20 --rounds 2 --cool 3 --dists normal "$@" 2>&1 | grep 'n=2' >> $out
for lib in "$@"; do
  ZF_LIB=$lib ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:fill_ctr -c 1 --csv python tools/prof_fill.py normal 32 1 2>/dev/null | grep dram__bytes >> $out
done
