# grid-waves sweep of the production fill (one library, one process per setting):
#   gpurun -- bash tools/ab_waves_sweep.sh lib.so "32:12 24 48 96" "28:6 12 24 48"
mkdir -p gpurun_out
LIB=$1; shift
out=gpurun_out/waves_sweep.txt
: > $out
for spec in "$@"; do
  n=${spec%%:*}
  for w in ${spec#*:}; do
    reps=$(( n >= 32 ? 3 : 20 ))
    echo "== n=2^$n waves $w" >> $out
    ZF_GRID_WAVES=$w python tools/ab.py --n $n --reps $reps --rounds 3 --cool 1 $LIB 2>&1 | grep '@1965' >> $out
  done
done
