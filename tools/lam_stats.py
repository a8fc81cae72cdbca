"""Per-config lambda agreement with the compiled reference: share of records
bit-identical, max and 99.99th percentile deviation in units of 2^-52 max|lambda|."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import paper_2511_00292_b200 as eig  # noqa: E402
from tests import _util as U  # noqa: E402

for cfg, lg in ((1, 20), (2, 22), (3, 22), (4, 22), (5, 22)):
    a_d = eig.generate(cfg, 1 << lg, seed=1000 + cfg)
    lam = eig.eigvals(a_d).lam.cpu().numpy()
    a = a_d.cpu().numpy()
    lam_r, _ = U.checker_eigvals(a, adv=False)
    same = U.bit_equal(lam, lam_r).all(axis=1)
    e = U.lam_error_units(lam, lam_r)
    fin = np.isfinite(e)
    print(f"config {cfg} (2^{lg}): bit-identical {100 * same.mean():.3f}%  max {e[fin].max():.2f} units  "
          f"p99.99 {np.percentile(e[fin], 99.99):.2f}  >4 units: {(e[fin] > 4).sum()}")
