"""Power/clock of the eigvals kernel vs. data-movement-only probes.

  python tools/power_memonly.py                      # product kernel
  TAG=memonly python tools/power_memonly.py         # eig33_probe_memonly: the same
                                                     # ring / tier tests / stores,
                                                     # no arithmetic
  TAG=stream python tools/power_memonly.py           # eig33_probe_stream: plain
                                                     # 72 B in / 24 B out stream

Prints median SM clock and board power (nvidia-smi, 50 ms) over ~3 s of
back-to-back launches on 2^27 config-3 records, and the record rate.
"""
import ctypes
import os
import statistics
import subprocess
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402

import paper_2511_00292_b200 as eig  # noqa: E402

L = eig.lib()
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), '..'))
import bench  # noqa: E402
PR = bench.probes_lib()  # measurement probes: tools/probes/libeig33_probes.so (not the product)


def sample(fn, secs=3.0):
    p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw",
                          "--format=csv,noheader,nounits", "-lms", "50"],
                         stdout=subprocess.PIPE, text=True)
    time.sleep(0.3)
    t0 = time.time()
    k = 0
    while time.time() - t0 < secs:
        fn()
        k += 1
    torch.cuda.synchronize()
    el = time.time() - t0
    p.terminate()
    rows = [ln.split(",") for ln in p.stdout.read().strip().splitlines() if "," in ln][6:]
    return (statistics.median(float(r[0]) for r in rows),
            statistics.median(float(r[1]) for r in rows), k / el)


def main():
    n = 1 << 27
    a = eig.generate(3, n, seed=1)
    lam = torch.empty((n, 3), dtype=torch.float64, device="cuda")
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    pa, pl = ctypes.c_void_p(a.data_ptr()), ctypes.c_void_p(lam.data_ptr())
    tag = os.environ.get("TAG", "product")
    if tag == "memonly":
        PR.eig33_probe_memonly.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_void_p]
        clk, pw, r = sample(lambda: PR.eig33_probe_memonly(pa, n, pl, st))
    elif tag == "stream":
        PR.eig33_probe_stream.argtypes = [ctypes.c_void_p, ctypes.c_longlong, ctypes.c_void_p,
                                         ctypes.c_void_p]
        clk, pw, r = sample(lambda: PR.eig33_probe_stream(pa, n, pl, st))
    else:
        clk, pw, r = sample(lambda: L.eig33cu_eigvals(pa, n, None, pl, None, st))
    print(f"{tag:10s} clk {clk:.0f} MHz power {pw:.0f} W  {r * n / 1e9:.1f} G rec/s"
          f"  -> {r * n * 96 / 1e12:.2f} TB/s")


if __name__ == "__main__":
    main()
