#!/bin/bash
for w in 1 4; do for p in 9 3 4; do for d in normal exp; do
  ZF_GRID_WAVES=$w ZF_PASS2=$p timeout 60 python tools/prof_fill.py $d 28 5 | sed "s|^|W$w P$p |"
done; done; done
