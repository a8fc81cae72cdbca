"""Throughput of the host-buffer path for PAGEABLE numpy buffers (what the
drop-in Python module sees) at large n: through eig.eigvals (fresh output array
per call, so its pages fault in during the call) and through
eig33_eigvals_host with a preallocated, already-touched output (pure staged
pipeline).  Run against a variant with EIG33_SO=... to compare builds.
  python tools/pageable_rate.py [log2_n ...]   (default 22 24)"""
import ctypes, os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np  # noqa: E402
import paper_2511_00292_b200 as eig  # noqa: E402

L = eig.lib()
P = lambda x: ctypes.c_void_p(x.ctypes.data)
tag = os.environ.get("TAG", "product")
for lg in [int(x) for x in sys.argv[1:]] or [22, 24]:
    n = 1 << lg
    a = np.ascontiguousarray(eig.generate(3, n, seed=3).cpu().numpy())
    lam = np.empty((n, 3))
    lam.fill(0.0)
    assert L.eig33_eigvals_host(P(a), n, None, P(lam), None, 0) == 0
    k = 5
    t0 = time.perf_counter()
    for _ in range(k):
        assert L.eig33_eigvals_host(P(a), n, None, P(lam), None, 0) == 0
    t1 = (time.perf_counter() - t0) / k
    eig.eigvals(a)
    t0 = time.perf_counter()
    for _ in range(k):
        eig.eigvals(a)
    t2 = (time.perf_counter() - t0) / k
    print(f"{tag:10s} n=2^{lg}: host ABI, touched output {n / t1 / 1e6:8.1f} M/s   eig.eigvals(numpy) {n / t2 / 1e6:8.1f} M/s",
          flush=True)
