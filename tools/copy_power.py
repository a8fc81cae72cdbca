"""Board power of a plain device-to-device copy (torch copy_, 4 GiB) of zeros vs
random doubles: how much of the data-movement energy depends on the bits moved."""
import os, statistics, subprocess, sys, time
import torch

N = 1 << 29  # doubles = 4 GiB
src = torch.empty(N, dtype=torch.float64, device="cuda")
dst = torch.empty_like(src)


def sample(secs=3.0):
    p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits",
                          "-lms", "50"], stdout=subprocess.PIPE, text=True)
    time.sleep(0.3)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.time()
    k = 0
    e0.record()
    while time.time() - t0 < secs:
        dst.copy_(src)
        k += 1
        if k % 8 == 0:
            torch.cuda.synchronize()
    e1.record()
    e1.synchronize()
    p.terminate()
    rows = [ln.split(",") for ln in p.stdout.read().strip().splitlines() if "," in ln][6:]
    gbs = k * 2 * N * 8 / (e0.elapsed_time(e1) * 1e-3) / 1e9
    return statistics.median(float(r[1]) for r in rows), statistics.median(float(r[0]) for r in rows), gbs


for name in ("zeros", "random"):
    if name == "zeros":
        src.zero_()
    else:
        src.copy_(torch.randn(N, dtype=torch.float64, device="cuda"))
    time.sleep(1.0)
    w, mhz, gbs = sample()
    print(f"copy {name:7s} {gbs:7.0f} GB/s  {w:6.0f} W  {mhz:5.0f} MHz  -> {(w - 258) / gbs * 1e3:6.1f} pJ/B above idle")
