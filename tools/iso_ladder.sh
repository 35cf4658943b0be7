# Cost-isolation ladder of the production fill (one GPU).  Build the variants
# first (here, nvcc cross-compiles):
#   python -c "from paper_1403_6870_b200 import _build as b; [b.build_variant(n, d) for n, d in
#     [('base', []), ('p2draw', ['ZF_DEBUG_P2=1']), ('p2store', ['ZF_DEBUG_P2=2']),
#      ('q1', ['ZF_DEBUG_Q=1']), ('q2', ['ZF_DEBUG_Q=2'])]]"
#   gpurun -- 'bash tools/iso_ladder.sh > gpurun_out/ladder.txt'
for i in 1 2; do
for lib in base p2draw p2store q1 q2; do
  for d in normal exp; do echo -n "$lib "; ZF_LIB=build/variants/$lib.so python tools/prof_fill.py $d 28 30; done
done
for d in normal exp; do echo -n "pass1only "; ZF_PASS2=9 ZF_LIB=build/variants/base.so python tools/prof_fill.py $d 28 30; done
done
