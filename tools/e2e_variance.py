"""Repeated end-to-end host-buffer runs (eig33_eigvals_host, 2^28 config-3 records,
pinned buffers) to check the e2e number is stable on a box."""
import ctypes, sys, time, torch
sys.path.insert(0, '/root/repo')
import paper_2511_00292_b200 as eig
L = eig.lib()
n = 1 << 28
a = eig.generate(3, n, seed=1)
h_a = torch.empty((n, 9), dtype=torch.float64, pin_memory=True); h_a.copy_(a)
h_l = torch.empty((n, 3), dtype=torch.float64, pin_memory=True)
del a; torch.cuda.empty_cache()
pa, pl = ctypes.c_void_p(h_a.data_ptr()), ctypes.c_void_p(h_l.data_ptr())
L.eig33_eigvals_host(pa, n, None, pl, None, 0)
for rep in range(6):
    t0 = time.perf_counter(); L.eig33_eigvals_host(pa, n, None, pl, None, 0); el = time.perf_counter() - t0
    print(f"e2e {n/el/1e9:.3f} G/s  H2D {n*72/el/1e9:.1f} GB/s")
