# ncu --set full of one normal 2^28 production fill per library build (source-level comparison):
#   gpurun -- bash tools/ncu_full_ab.sh name1=lib1.so name2=lib2.so ...
mkdir -p gpurun_out
for kv in "$@"; do
  name=${kv%%=*}; lib=${kv#*=}
  ZF_LIB=$lib ncu --set full --import-source on --clock-control none -k regex:fill_ctr_kernel -c 1 \
      -o gpurun_out/abfull_$name -f python tools/prof_fill.py ${DIST:-normal} 28 1 > gpurun_out/abfull_$name.log 2>&1
done
