# A/B library builds on f64/f32 fills and the generate-and-sum kernel (one GPU)
for i in 1 2; do
  for lib in "$@"; do
    for d in normal exp; do
      for t in f64 f32; do echo -n "$(basename $lib) $t "; ZF_LIB=$lib python tools/prof_fill.py $d 28 30 $t; done
    done
    echo -n "$(basename $lib) agg "; ZF_LIB=$lib python tools/bench_configs.py agg | head -2 | tr '\n' ' '; echo
  done
done
