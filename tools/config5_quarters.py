"""lambda throughput of each quarter of config 5 (2^22 records): q0 near-scalar,
q1 exact repeated eigenvalues, q2 diagonal, q3 2^k-scaled (k in [-500, 500])."""
import ctypes, os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402
import paper_2511_00292_b200 as eig  # noqa: E402

L = eig.lib()
P = lambda t: ctypes.c_void_p(t.data_ptr())
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
tag = os.environ.get("TAG", "product")
n = 1 << 22
a = eig.generate(5, n, seed=105)
q = n // 4
for k in range(4):
    aq = a[k * q:(k + 1) * q].contiguous()
    lam = torch.empty((q, 3), dtype=torch.float64, device="cuda")
    for name, fl in (("lam", None), ("lam+flags", torch.empty(q, dtype=torch.uint8, device="cuda"))):
        fn = lambda: L.eig33cu_eigvals(P(aq), q, None, P(lam), None if fl is None else P(fl), st)
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
        print(f"{tag:10s} config 5 q{k} {name:10s} {q / t / 1e9:6.2f} G rec/s")
