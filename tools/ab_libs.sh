# A/B several library builds on the production fill (one GPU), interleaved:
#   gpurun -- bash tools/ab_libs.sh build/variants/a.so build/variants/b.so ...
for i in 1 2 3; do
  for lib in "$@"; do
    for d in normal exp; do echo -n "$(basename $lib) "; ZF_LIB=$lib python tools/prof_fill.py $d 28 30; done
  done
done
