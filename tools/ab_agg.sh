# A/B library builds on the generate-and-sum (aggregate) kernel:
#   gpurun -- bash tools/ab_agg.sh build/variants/a.so build/variants/b.so
for i in 1 2; do for lib in "$@"; do echo -n "$(basename $lib) "; ZF_LIB=$lib python tools/bench_configs.py agg; done; done
