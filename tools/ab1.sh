python tools/power_probe.py 28 3 normal > gpurun_out/power_normal.txt 2>&1
sleep 5
python tools/power_probe.py 28 2 fill_ > gpurun_out/power_fill.txt 2>&1
