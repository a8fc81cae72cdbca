"""Where a k_fused launch spends its time (diagnostic build EIG33_TIMELINE=1):
per-warp %globaltimer at entry, after griddepcontrol.wait, first chunk landed,
and exit, for back-to-back launches of config-3 batches of several sizes.

  python -c "from paper_2511_00292_b200 import build; build.build_variant('timeline', ['EIG33_TIMELINE=1'])"
  EIG33_SO=paper_2511_00292_b200/build/variants/timeline.so python tools/timeline.py
"""
import ctypes, os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import paper_2511_00292_b200 as eig  # noqa: E402

L = eig.lib()
L.eig33_debug_timeline.argtypes = [ctypes.c_void_p, ctypes.c_int]
P = lambda t: ctypes.c_void_p(t.data_ptr())
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
W = 148 * 2 * 8
for lg in (18, 20, 22):
    n = 1 << lg
    a = eig.generate(3, n, seed=7)
    lam = torch.empty((n, 3), dtype=torch.float64, device="cuda")
    for _ in range(5):
        assert L.eig33cu_eigvals(P(a), n, None, P(lam), None, st) == 0
    torch.cuda.synchronize()
    tl = np.zeros((W, 4), np.uint64)
    assert L.eig33_debug_timeline(tl.ctypes.data, W) == 0
    nw = min(W, (n + 63) // 64)
    if os.environ.get("TL_SAVE"):
        np.save(os.path.join(os.environ["TL_SAVE"], f"timeline_2p{lg}.npy"), tl[:nw])
    t = tl[:nw].astype(np.int64)
    t0 = t[:, 0].min()
    rel = (t - t0) / 1e3  # us
    span = rel[:, 3].max()
    print(f"n=2^{lg}: launch span {span:7.2f} us | entry  min {rel[:,0].min():6.2f} max {rel[:,0].max():6.2f} | "
          f"after-wait med {np.median(rel[:,1]):6.2f} max {rel[:,1].max():6.2f} | first-chunk med "
          f"{np.median(rel[:,2]):6.2f} max {rel[:,2].max():6.2f} | exit min {rel[:,3].min():6.2f} "
          f"med {np.median(rel[:,3]):6.2f} max {rel[:,3].max():6.2f} | ideal {n / 45e9 * 1e6:6.2f} us")
