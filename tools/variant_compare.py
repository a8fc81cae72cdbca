"""Compact A/B measurement of a build (EIG33_SO=... selects it): lambda and
lambda+inv+flags rates on every BASELINE config at its size, config 3 at
2^20 / 2^22 / 2^26, and config 5's quarters; burst rates (20 launches after 3
warm-ups, CUDA events, 0.5 s idle before each).  One line per number:
  TAG  name  G_records/s"""
import ctypes, os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402
import paper_2511_00292_b200 as eig  # noqa: E402

L = eig.lib()
P = lambda t: None if t is None else ctypes.c_void_p(t.data_ptr())
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
tag = os.environ.get("TAG", "product")


def rate(fn, n, reps=20):
    torch.cuda.synchronize()
    time.sleep(0.5)
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return n / (e0.elapsed_time(e1) / reps * 1e-3) / 1e9


ONLY = [c for c in os.environ.get("VC_CASES", "").split(",") if c]  # e.g. VC_CASES=c4,c5_q0


def case(cfg, n, first=0, name=None):
    if ONLY and (name or f"c{cfg}") not in ONLY:
        return
    a = eig.generate(cfg, n, seed=100 + cfg, first_index=first)
    lam = torch.empty((n, 3), dtype=torch.float64, device="cuda")
    inv = torch.empty((n, 4), dtype=torch.float64, device="cuda")
    fl = torch.empty((n,), dtype=torch.uint8, device="cuda")
    nm = name or f"c{cfg}"
    r1 = rate(lambda: L.eig33cu_eigvals(P(a), n, None, P(lam), None, st), n)
    r2 = rate(lambda: L.eig33cu_eigvals(P(a), n, P(inv), P(lam), P(fl), st), n)
    print(f"{tag:10s} {nm:14s} lam {r1:6.2f}   full {r2:6.2f}", flush=True)


case(3, 1 << 20, name="c3_2^20")
case(3, 1 << 22, name="c3_2^22")
case(3, 1 << 26, name="c3_2^26")
case(1, 1 << 20)
case(2, 1 << 22)
case(4, 1 << 22)
case(5, 1 << 22)
for q in range(4):
    case(5, 1 << 20, first=q << 20, name=f"c5_q{q}")
