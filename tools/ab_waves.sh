# grid-size sweep of the production fill (ZF_GRID_WAVES = resident waves per launch)
for i in 1 2; do for w in ${WAVES:-1 2 3 4 6 8 16}; do
  for d in normal exp; do echo -n "waves=$w "; ZF_GRID_WAVES=$w python tools/prof_fill.py $d 28 30; done
done; done
