"""Run eig33cu_eigvals on one BASELINE config a few times (for ncu captures):
  python tools/run_config.py CONFIG [log2_n=22] [reps=3] [flags=0] [first_index=0] [inv=0]"""
import ctypes, os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402
import paper_2511_00292_b200 as eig  # noqa: E402

cfg = int(sys.argv[1])
n = 1 << (int(sys.argv[2]) if len(sys.argv) > 2 else 22)
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
want_flags = len(sys.argv) > 4 and sys.argv[4] == "1"
first = int(sys.argv[5]) if len(sys.argv) > 5 else 0
want_inv = len(sys.argv) > 6 and sys.argv[6] == "1"
L = eig.lib()
P = lambda t: None if t is None else ctypes.c_void_p(t.data_ptr())
a = eig.generate(cfg, n, seed=100 + cfg, first_index=first)
lam = torch.empty((n, 3), dtype=torch.float64, device="cuda")
fl = torch.empty((n,), dtype=torch.uint8, device="cuda") if want_flags else None
inv = torch.empty((n, 4), dtype=torch.float64, device="cuda") if want_inv else None
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
for _ in range(reps):
    assert L.eig33cu_eigvals(P(a), n, P(inv), P(lam), P(fl), st) == 0
torch.cuda.synchronize()
print("ok")
