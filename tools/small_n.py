"""Fixed per-launch overhead of k_fused: config-3 lambda throughput vs batch size
(20 launches after 3 warm-ups, CUDA events).  TAG / EIG33_SO select a build."""
import ctypes, os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402
import paper_2511_00292_b200 as eig  # noqa: E402

L = eig.lib()
P = lambda t: ctypes.c_void_p(t.data_ptr())
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
tag = os.environ.get("TAG", "product")
for lg in (16, 18, 20, 22, 24, 26):
    n = 1 << lg
    a = eig.generate(3, n, seed=7)
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
    print(f"{tag:8s} n=2^{lg:2d}  {t * 1e6:9.1f} us  {n / t / 1e9:6.2f} G rec/s")
