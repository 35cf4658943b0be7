#!/bin/bash
# usage: tools/variants.sh "<policies>" <libs...>   (runs prof_fill per lib x policy x dist)
pols="$1"; shift
for lib in "$@"; do
  for p in $pols; do
    for d in normal exp; do
      ZF_LIB=$lib ZF_PASS2=$p timeout 60 python tools/prof_fill.py $d 28 5 | sed "s|^|$(basename $lib) P$p |"
    done
  done
done
