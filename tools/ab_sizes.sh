# A/B library builds at several fill sizes (normal and exp, fp64)
for i in 1 2; do for lg in ${SIZES:-26 28 32}; do for lib in $LIBS; do
  for d in normal exp; do echo -n "$(basename $lib) n=2^$lg "; ZF_LIB=$lib python tools/prof_fill.py $d $lg $(( lg > 30 ? 4 : 20 )); done
done; done; done
