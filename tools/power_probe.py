"""Sustained-load clock / power probe (experiment tool): runs fills back to back
for a few seconds and samples NVML every ~20 ms."""
import sys, time, threading
sys.path.insert(0, ".")
import torch
import pynvml as N
import paper_1403_6870_b200 as zf

N.nvmlInit()
h = N.nvmlDeviceGetHandleByIndex(0)
rows = []
stop = threading.Event()
def samp():
    while not stop.is_set():
        r = N.nvmlDeviceGetCurrentClocksEventReasons(h)
        rows.append((time.perf_counter(), N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM),
                     N.nvmlDeviceGetPowerUsage(h) / 1000.0, N.nvmlDeviceGetTemperature(h, 0), r))
        time.sleep(0.02)
n = 1 << int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 28
secs = float(sys.argv[2]) if len(sys.argv) > 2 else 3.0
what = sys.argv[3] if len(sys.argv) > 3 else "normal"
out = torch.empty(n, dtype=torch.float64, device="cuda")
s = (zf.NormalSampler if what == "normal" else zf.ExpSampler)(source=zf.UniformSource.counter(7))
t = threading.Thread(target=samp, daemon=True); t.start()
t0 = time.perf_counter(); k = 0
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
while time.perf_counter() - t0 < secs:
    if what == "fill_":
        out.fill_(1.0)
    else:
        s.fill(out)
    k += 1
    if k % 20 == 0:
        torch.cuda.synchronize()
torch.cuda.synchronize()
stop.set(); t.join()
dt = time.perf_counter() - t0
print(f"{what} n=2^{n.bit_length()-1}: {k} launches in {dt:.2f}s = {k*n/dt/1e9:.1f} G/s avg")
for r in rows[::5]:
    print(f"t={r[0]-t0:6.3f} sm={r[1]} W={r[2]:.0f} T={r[3]} reasons=0x{r[4]:x}")
