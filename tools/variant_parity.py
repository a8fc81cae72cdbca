"""Parity of an experimental build (EIG33_SO=...) against the compiled
reference on ragged sizes of configs 1-5: invariants (fused and invariants-only
entry points) and flags bitwise, lambda through the suite's gate.
  EIG33_SO=paper_2511_00292_b200/build/variants/<name>.so python tools/variant_parity.py"""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402
import paper_2511_00292_b200 as eig  # noqa: E402
from tests import _util as U  # noqa: E402

so = os.environ.get("EIG33_SO", "product")
for n in (1, 63, 64, 65, 4096 * 32 + 7, (1 << 20) + 33, (1 << 22) + 1):
    for cfg in (1, 2, 3, 4, 5):
        a = eig.generate(cfg, n, seed=n + cfg)
        r = eig.eigvals(a, return_invariants=True, return_flags=True)
        inv_only = eig.invariants(a)
        torch.cuda.synchronize()
        an = a.cpu().numpy()
        inv_r = U.checker_invariants(an)
        lam_r, adv_r = U.checker_eigvals(an)
        assert U.bit_equal(r.inv.cpu().numpy(), inv_r).all(), (n, cfg)
        assert U.bit_equal(inv_only.cpu().numpy(), inv_r).all(), (n, cfg)
        assert ((r.flags.cpu().numpy() & 1) == adv_r).all(), (n, cfg, "flags")
        U.lam_gate(an, r.lam.cpu().numpy(), lam_r, inv_ref=inv_r)
print("variant parity ok", so)
