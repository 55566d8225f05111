"""SM clock, power draw and throttle reasons while a Dense-chain training step
runs back to back (tools only): is the step power-bound?

  python tools/power_probe.py WIDTH DEPTH BATCH [seconds]
"""
import statistics
import sys
import threading
import time

import numpy as np
import pynvml
import torch

from paper_1811_01457_b200.dense import Chain, Dense
from paper_1811_01457_b200.train import Trainer

width, depth, batch = (int(v) for v in sys.argv[1:4])
secs = float(sys.argv[4]) if len(sys.argv) > 4 else 3.0
acts = ("tanh",) * (depth - 1) + ("identity",)
chain = Chain(*[Dense(width, width, a) for a in acts]).init_params(np.random.default_rng(0))
tr = Trainer(chain, batch, loss="mse", lr=1e-4, precision="bf16", graph=True)
X = torch.rand((batch, width), device="cuda")
Y = torch.rand((batch, width), device="cuda") * 2 - 1
for _ in range(5):
    tr.step(X, Y)
torch.cuda.synchronize()
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
samples, stop = [], threading.Event()


def sample():
    while not stop.is_set():
        samples.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                        pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0,
                        pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)))
        time.sleep(0.005)


t = threading.Thread(target=sample, daemon=True)
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t.start()
t0 = time.time()
n = 0
s.record()
while time.time() - t0 < secs:
    for _ in range(20):
        tr.step(X, Y)
    n += 20
    torch.cuda.synchronize()
e.record()
torch.cuda.synchronize()
stop.set()
t.join()
ms = s.elapsed_time(e) / n
load = samples[len(samples) // 10:]
mhz = statistics.median(x[0] for x in load)
watts = statistics.median(x[1] for x in load)
pcap = sum(1 for x in load if x[2] & 0x4) / max(1, len(load))
limit = pynvml.nvmlDeviceGetEnforcedPowerLimit(h) / 1000.0
print(f"{width}x{depth} batch {batch}: {ms:.4f} ms/step over {n} steps; SM {mhz:.0f} MHz median, "
      f"power {watts:.0f} W median (limit {limit:.0f} W), sw_power_cap in {pcap * 100:.0f} % of samples")
