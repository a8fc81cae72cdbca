# quick parity of split-tail builds against the product build on ragged sizes
import os, sys, ctypes
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2511_00292_b200 as eig
from tests import _util as U
so = os.environ["EIG33_SO"]
for n in (1, 63, 64, 65, 4096 * 32 + 7, (1 << 20) + 33, (1 << 22) + 1):
    for cfg in (3, 5):
        a = eig.generate(cfg, n, seed=n + cfg)
        r = eig.eigvals(a, return_invariants=True, return_flags=True)
        inv_only = eig.invariants(a)
        torch.cuda.synchronize()
        an = a.cpu().numpy()
        inv_r = U.checker_invariants(an); lam_r, adv_r = U.checker_eigvals(an)
        assert U.bit_equal(r.inv.cpu().numpy(), inv_r).all(), (n, cfg)
        assert U.bit_equal(inv_only.cpu().numpy(), inv_r).all(), (n, cfg)
        assert ((r.flags.cpu().numpy() & 1) == adv_r).all(), (n, cfg)
        U.lam_gate(an, r.lam.cpu().numpy(), lam_r, inv_ref=inv_r)
print("split parity ok", so)
