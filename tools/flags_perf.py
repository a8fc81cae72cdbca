"""lambda+flags and lambda+inv+flags throughput on configs 4 and 5 and config 5's
near-scalar quarter (advisory-heavy), 20 launches after 1 s idle."""
import ctypes, os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402
import paper_2511_00292_b200 as eig  # noqa: E402

L = eig.lib()
P = lambda t: None if t is None else ctypes.c_void_p(t.data_ptr())
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
tag = os.environ.get("TAG", "product")
n = 1 << 22
for name, a in (("config4", eig.generate(4, n, seed=104)), ("config5", eig.generate(5, n, seed=105)),
                ("config5-q0", eig.generate(5, n, seed=105)[: n // 4].contiguous())):
    m = a.shape[0]
    lam = torch.empty((m, 3), dtype=torch.float64, device="cuda")
    inv = torch.empty((m, 4), dtype=torch.float64, device="cuda")
    fl = torch.empty((m,), dtype=torch.uint8, device="cuda")
    for what, iv in (("lam+flags", None), ("lam+inv+flags", inv)):
        fn = lambda: L.eig33cu_eigvals(P(a), m, P(iv), P(lam), P(fl), st)
        torch.cuda.synchronize()
        time.sleep(1.0)
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
        print(f"{tag:10s} {name:11s} {what:14s} {m / t / 1e9:6.2f} G rec/s")
