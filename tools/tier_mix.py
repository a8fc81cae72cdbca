"""Which k_fused tier each 32-record warp step of a BASELINE config takes:
steady (all moderate, J2 > 0, disc > 0), moderate (all moderate, some J2 <= 0
or disc <= 0) or general (some record outside [2^-100, 2^100) or non-finite)."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np  # noqa: E402
import paper_2511_00292_b200 as eig  # noqa: E402

n = 1 << 22
for cfg in (1, 2, 3, 4, 5):
    a = eig.generate(cfg, n, seed=100 + cfg)
    inv = eig.invariants(a).cpu().numpy()
    h = a.cpu().numpy()
    e = (h.view(np.uint64) >> np.uint64(52)) & np.uint64(0x7FF)
    ok = (h == 0) | ((e >= 1023 - 100) & (e < 1023 + 100))  # is_moderate: [2^-100, 2^100)
    mod = ok.all(axis=1)
    fast = mod & (inv[:, 1] > 0) & (inv[:, 3] > 0)
    w_mod = mod.reshape(-1, 32).all(axis=1)
    w_fast = fast.reshape(-1, 32).all(axis=1)
    print(f"config {cfg}: records non-moderate {100 * (1 - mod.mean()):6.2f}%  not-steady {100 * (1 - fast.mean()):6.2f}% | "
          f"warp steps steady {100 * w_fast.mean():6.2f}%  moderate {100 * (w_mod & ~w_fast).mean():6.2f}%  "
          f"general {100 * (~w_mod).mean():6.2f}%")
