"""lambda-only throughput of configs 3 and 4 (2^22 records, 20 launches after 3
warm-ups) -- config 3 runs the steady tier, config 4 the moderate tier."""
import ctypes, os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402
import paper_2511_00292_b200 as eig  # noqa: E402

L = eig.lib()
P = lambda t: ctypes.c_void_p(t.data_ptr())
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
tag = os.environ.get("TAG", "product")
n = 1 << 22
for cfg in (3, 4, 5):
    a = eig.generate(cfg, n, seed=100 + cfg)
    lam = torch.empty((n, 3), dtype=torch.float64, device="cuda")
    fn = lambda: L.eig33cu_eigvals(P(a), n, None, P(lam), None, st)
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        fn()
    e1.record()
    e1.synchronize()
    t = e0.elapsed_time(e1) / 20 * 1e-3
    print(f"{tag:14s} config {cfg}  {n / t / 1e9:6.2f} G rec/s")
