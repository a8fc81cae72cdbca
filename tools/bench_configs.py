"""Throughput of every entry point on every BASELINE config at its batch size
(supplementary to bench.py, whose line is config 3 / lambda only).  CUDA-event
timing, device-resident inputs, 20 timed launches after 3 warm-ups, each
measurement after 1 s idle so that the previous one's power-capped clocks do
not carry over (short runs: these are burst rates, above the sustained
power-capped rate of bench.py)."""
import ctypes, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2511_00292_b200 as eig

L = eig.lib()
SIZES = {1: 1 << 20, 2: 1 << 22, 3: 1 << 26, 4: 1 << 22, 5: 1 << 22}
P = lambda t: None if t is None else ctypes.c_void_p(t.data_ptr())


def timeit(fn, reps=20, warm=3):
    torch.cuda.synchronize()
    time.sleep(1.0)
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


rows = []
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
for cfg, n in SIZES.items():
    a = eig.generate(cfg, n, seed=100 + cfg)
    lam = torch.empty((n, 3), dtype=torch.float64, device="cuda")
    inv = torch.empty((n, 4), dtype=torch.float64, device="cuda")
    fl = torch.empty((n,), dtype=torch.uint8, device="cuda")
    cases = {
        "eigvals lam": lambda: L.eig33cu_eigvals(P(a), n, None, P(lam), None, st),
        "eigvals lam+inv+flags": lambda: L.eig33cu_eigvals(P(a), n, P(inv), P(lam), P(fl), st),
        "invariants": lambda: L.eig33cu_invariants(P(a), n, P(inv), st),
    }
    if cfg == 1:
        cases["eigvalss lam+flags"] = lambda: L.eig33cu_eigvalss(P(a), n, None, P(lam), P(fl), st)
    for name, fn in cases.items():
        t = timeit(fn)
        rows.append({"config": cfg, "n": n, "entry": name, "G_records_per_s": n / t / 1e9})
        print(f"config {cfg}  n={n:>9d}  {name:24s} {n / t / 1e9:7.2f} G records/s")
    del a, lam, inv, fl
print(json.dumps(rows))
