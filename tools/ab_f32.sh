# A/B library builds on fp32 and fp64 production fills (one GPU), interleaved
for i in 1 2 3; do
  for lib in "$@"; do
    for d in normal exp; do
      for t in f64 f32; do echo -n "$(basename $lib) $t "; ZF_LIB=$lib python tools/prof_fill.py $d 28 30 $t; done
    done
  done
done
