"""Wall-clock latency of single-matrix and small-batch calls through the
drop-in module and the host-buffer C ABI (GPU round trip per call)."""
import os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np  # noqa: E402
import paper_2511_00292_b200 as eig  # noqa: E402
from paper_2511_00292_b200 import eig33  # noqa: E402

m = [[2, 1, 0], [1, 3, -1], [0, -1, 4]]
for _ in range(20):
    eig33.eigvals(m)
for name, fn in (("eig33.eigvals(3x3 list)", lambda: eig33.eigvals(m)),
                 ("eig33.j2_stable(3x3 list)", lambda: eig33.j2_stable(m))):
    t0 = time.perf_counter()
    k = 200
    for _ in range(k):
        fn()
    print(f"{name:28s} {(time.perf_counter() - t0) / k * 1e6:8.1f} us/call")
for n in (1, 64, 4096, 1 << 16, 1 << 20, 1 << 22):
    a = np.random.default_rng(n).standard_normal((n, 9))
    eig.eigvals(a)
    k = max(3, min(200, (1 << 22) // n))
    t0 = time.perf_counter()
    for _ in range(k):
        eig.eigvals(a)
    dt = (time.perf_counter() - t0) / k
    print(f"eigvals(host (n,9)) n={n:8d}  {dt * 1e6:9.1f} us/call  {n / dt / 1e6:9.2f} M records/s")
