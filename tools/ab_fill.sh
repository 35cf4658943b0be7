# A/B of two library builds on the production fill (one GPU):
#   python -c "from paper_1403_6870_b200 import _build; _build.build_variant('old', [])"
#   gpurun -- bash tools/ab_fill.sh [build/variants/old.so]
OLD=${1:-build/variants/old.so}
for i in 1 2 3; do
  for lib in $OLD paper_1403_6870_b200/libzigfast_b200.so; do
    for d in normal exp; do echo -n "$lib "; ZF_LIB=$lib python tools/prof_fill.py $d 28 30; done
    for d in normal exp; do echo -n "$lib "; ZF_LIB=$lib python tools/prof_fill.py $d 28 30 f32; done
  done
done
