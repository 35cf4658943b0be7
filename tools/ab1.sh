V=build/variants
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/r2_gputests.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_gputests.txt
timeout 300 python tools/ab.py --cool 0.15 --n 28 --reps 6 --rounds 8 $V/cur.so $V/spec2.so > gpurun_out/ab8_28.txt 2>&1
timeout 300 python tools/ab.py --cool 0.3 --n 32 --reps 1 --rounds 6 $V/cur.so $V/spec2.so > gpurun_out/ab8_32.txt 2>&1
