"""Throughput by output mix (lam / lam+inv / lam+inv+flags / inv only), burst
timing (20 launches after 3 warm-ups); config 3 at 2^26 records by default
(SM_CONFIG=c, SM_LOG2N=k select another).  Run against a variant with
EIG33_SO=... to compare builds."""
import ctypes, os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402
import paper_2511_00292_b200 as eig  # noqa: E402

L = eig.lib()
P = lambda t: None if t is None else ctypes.c_void_p(t.data_ptr())
cfg = int(os.environ.get("SM_CONFIG", "3"))
n = 1 << int(os.environ.get("SM_LOG2N", "26"))
a = eig.generate(cfg, n, seed=100 + cfg)
lam = torch.empty((n, 3), dtype=torch.float64, device="cuda")
inv = torch.empty((n, 4), dtype=torch.float64, device="cuda")
fl = torch.empty((n,), dtype=torch.uint8, device="cuda")
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def timeit(fn, reps=20, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps * 1e-3


tag = os.environ.get("TAG", "product")
for name, fn, b in [
    ("lam", lambda: L.eig33cu_eigvals(P(a), n, None, P(lam), None, st), 96),
    ("lam+flags", lambda: L.eig33cu_eigvals(P(a), n, None, P(lam), P(fl), st), 97),
    ("lam+inv", lambda: L.eig33cu_eigvals(P(a), n, P(inv), P(lam), None, st), 128),
    ("lam+inv+flags", lambda: L.eig33cu_eigvals(P(a), n, P(inv), P(lam), P(fl), st), 129),
    ("inv", lambda: L.eig33cu_invariants(P(a), n, P(inv), st), 104),
    ("sym lam", lambda: L.eig33cu_eigvalss(P(a), n, None, P(lam), None, st), 96),
    ("sym lam+inv+fl", lambda: L.eig33cu_eigvalss(P(a), n, P(inv), P(lam), P(fl), st), 129),
]:
    t = timeit(fn)
    print(f"{tag:10s} c{cfg} {name:14s} {n / t / 1e9:6.2f} G rec/s  {n * b / t / 1e12:5.2f} TB/s")
