V=build/variants
ZF_PASS2=9 timeout 900 python tools/ab.py --no-check --sustain 2.0 --rounds 1 --n 30 --dists normal $V/cur.so $V/p1d1.so $V/p1d2.so $V/p1d3.so $V/p1d4.so > gpurun_out/ab16_energy.txt 2>&1
ZF_PASS2=9 timeout 300 python tools/ab.py --no-check --cool 0.15 --n 28 --reps 6 --rounds 4 --dists normal $V/cur.so $V/p1d1.so $V/p1d2.so $V/p1d3.so $V/p1d4.so > gpurun_out/ab16_cold.txt 2>&1
