"""Small workload touching every kernel and code path (TMA ring, ragged tails,
misaligned coalesced path, advisory, eigvalss, study kernels, generator) for
compute-sanitizer runs.  Exits 0 on success."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2511_00292_b200 as eig
from tests import _util as U

for n in (1, 33, 64, 65, 1000, 4099):
    a = torch.from_numpy(U.mixed_corpus(max(n, 8), n)[:n]).cuda()
    eig.eigvals(a, return_invariants=True, return_flags=True)
    eig.eigvalss(a, return_invariants=True, return_flags=True)
    eig.invariants(a)
    buf = torch.empty(n * 9 + 1, dtype=torch.float64, device="cuda")
    buf[1:] = a.reshape(-1)
    eig.eigvals(buf[1:].view(n, 9), return_flags=True)
for cfg in range(1, 6):
    g = eig.generate(cfg, 3000, seed=cfg)
    eig.eigvals(g, return_flags=True)
# many chunks per block (dynamic chunk counter) with a ragged last chunk, and an
# invariants output that is not 32-B aligned (scalar-store path)
import ctypes  # noqa: E402
L = eig.lib()
for n in ((3 << 20) + 5, 100003):
    g = eig.generate(5, n, seed=7)
    lam = torch.empty((n, 3), dtype=torch.float64, device="cuda")
    invb = torch.empty(n * 4 + 1, dtype=torch.float64, device="cuda")
    fl = torch.empty(n, dtype=torch.uint8, device="cuda")
    P = lambda t: ctypes.c_void_p(t.data_ptr())
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    assert L.eig33cu_eigvals(P(g), n, ctypes.c_void_p(invb.data_ptr() + 8), P(lam), P(fl), st) == 0
    assert L.eig33cu_invariants(P(g), n, ctypes.c_void_p(invb.data_ptr() + 8), st) == 0
    torch.cuda.synchronize()
j3 = torch.randn(1000, dtype=torch.float64, device="cuda")
eig.triple_angle(j3, torch.randn(1000, dtype=torch.float64, device="cuda"))
a = U.mixed_corpus(2000, 3)
eig.invariants(a, variant="Naive")
eig.invariants(a, variant="NaiveTensor")
eig.eigvals_naive(a, return_flags=True)
eig.jacobians(a)
eig.eigvals(a)  # host pipeline (pageable, direct)
eig.disc_naive(j3, torch.randn(1000, dtype=torch.float64, device="cuda"))
big = U.mixed_corpus((1 << 17) + 7, 4)  # >= 8 MB pageable: staged pinned-bounce pipeline
eig.eigvals(big, return_invariants=True, return_flags=True)
eig.invariants(big)
from paper_2511_00292_b200 import eig33  # noqa: E402
eig33.eigvals([[2, 1, 0], [1, 3, -1], [0, -1, 4]])
eig33.jacobian_disc([1, 2, 3, 4, 5, 6, 7, 8, 10])
torch.cuda.synchronize()
print("sanitize smoke ok")
