"""Launch eig33cu_eigvals once per case, for ncu captures of several workloads
in one process:  python tools/run_cases.py CASE [CASE ...]
CASE = config:log2n[:first_index[:full]]   (full=1: invariants + flags too)"""
import ctypes, os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402
import paper_2511_00292_b200 as eig  # noqa: E402

L = eig.lib()
P = lambda t: None if t is None else ctypes.c_void_p(t.data_ptr())
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
for spec in sys.argv[1:]:
    f = spec.split(":")
    cfg, n = int(f[0]), 1 << int(f[1])
    first = int(f[2]) if len(f) > 2 else 0
    full = len(f) > 3 and f[3] == "1"
    a = eig.generate(cfg, n, seed=100 + cfg, first_index=first)
    lam = torch.empty((n, 3), dtype=torch.float64, device="cuda")
    inv = torch.empty((n, 4), dtype=torch.float64, device="cuda") if full else None
    fl = torch.empty((n,), dtype=torch.uint8, device="cuda") if full else None
    assert L.eig33cu_eigvals(P(a), n, P(inv), P(lam), P(fl), st) == 0
    torch.cuda.synchronize()
print("ok")
