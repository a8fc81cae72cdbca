"""Median power / SM clock (nvidia-smi, 50 ms) while running, for ~3 s each:
the FP64 DFMA probe, an HBM copy, and the fused kernel on config 3."""
import ctypes, os, statistics, subprocess, sys, threading, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2511_00292_b200 as eig

L = eig.lib()
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), '..'))
import bench  # noqa: E402
PR = bench.probes_lib()  # measurement probes: tools/probes/libeig33_probes.so (not the product)


def sample(fn, secs=3.0):
    p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits",
                          "-lms", "50"], stdout=subprocess.PIPE, text=True)
    time.sleep(0.3)
    t0 = time.time()
    n = 0
    while time.time() - t0 < secs:
        fn()
        n += 1
    torch.cuda.synchronize()
    el = time.time() - t0
    p.terminate()
    rows = [l.split(",") for l in p.stdout.read().strip().splitlines() if "," in l]
    rows = rows[len(rows) // 4:]
    clk = statistics.median(float(r[0]) for r in rows)
    pw = statistics.median(float(r[1]) for r in rows)
    return clk, pw, n / el


PR.eig33_probe_fp64_op.restype = ctypes.c_double
PR.eig33_probe_fp64_op.argtypes = [ctypes.c_int] * 3
print("dfma    clk %.0f MHz  power %.0f W  calls/s %.1f" % sample(lambda: PR.eig33_probe_fp64_op(0, 20, 8192)))
x = torch.empty(1 << 31, dtype=torch.uint8, device="cuda")
y = torch.empty_like(x)
clk, pw, r = sample(lambda: y.copy_(x))
print("copy    clk %.0f MHz  power %.0f W  GB/s %.0f" % (clk, pw, r * 2 * (1 << 31) / 1e9))
del x, y
n = 1 << 27
a = eig.generate(3, n, seed=1)
lam = torch.empty((n, 3), dtype=torch.float64, device="cuda")
st = torch.cuda.current_stream().cuda_stream
clk, pw, r = sample(lambda: L.eig33cu_eigvals(ctypes.c_void_p(a.data_ptr()), n, None, ctypes.c_void_p(lam.data_ptr()), None, ctypes.c_void_p(st)))
print("eig33   clk %.0f MHz  power %.0f W  G rec/s %.1f" % (clk, pw, r * n / 1e9))
time.sleep(2)
def idle():
    time.sleep(0.05)
print("idle    clk %.0f MHz  power %.0f W" % sample(idle)[:2])
n2 = 1 << 20
a2 = a[:n2].clone()
l2 = torch.empty((n2, 3), dtype=torch.float64, device="cuda")
clk, pw, r = sample(lambda: L.eig33cu_eigvals(ctypes.c_void_p(a2.data_ptr()), n2, None, ctypes.c_void_p(l2.data_ptr()), None, ctypes.c_void_p(st)))
print("eig33-L2resident clk %.0f MHz  power %.0f W  G rec/s %.1f" % (clk, pw, r * n2 / 1e9))
inv = torch.empty((n, 4), dtype=torch.float64, device="cuda")
clk, pw, r = sample(lambda: L.eig33cu_invariants(ctypes.c_void_p(a.data_ptr()), n, ctypes.c_void_p(inv.data_ptr()), ctypes.c_void_p(st)))
print("inv-only clk %.0f MHz  power %.0f W  G rec/s %.1f" % (clk, pw, r * n / 1e9))
