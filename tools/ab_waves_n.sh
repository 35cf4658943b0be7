# grid-size sweep across fill sizes (normal and exp, fp64)
for lg in ${SIZES:-26 28 30 32}; do for w in ${WAVES:-4 6 8 12 16}; do
  for d in normal exp; do echo -n "n=2^$lg waves=$w "; ZF_GRID_WAVES=$w python tools/prof_fill.py $d $lg $(( lg > 30 ? 4 : 20 )); done
done; done
