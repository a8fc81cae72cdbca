"""Long GPU parity fuzz (not part of the test suite): many seeded batches of
random bit patterns, mixed corpora, moderate-range edges and generated configs
through eig33cu_eigvals (invariants + flags) and eig33cu_eigvalss, each checked
against the compiled reference with the test suite's own gates.
  python tools/fuzz_gpu.py [batches=8] [log2_records=22] [first_batch=0]"""
import os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import paper_2511_00292_b200 as eig  # noqa: E402
from tests import _util as U  # noqa: E402
from tests.test_hostmath import _moderate_edge_corpus  # noqa: E402
from tests.test_parity_gpu import _assert_parity  # noqa: E402
from tests import _exact  # noqa: E402


def run(a):
    r = eig.eigvals(torch.from_numpy(a).cuda(), return_invariants=True, return_flags=True)
    torch.cuda.synchronize()
    return r.lam.cpu().numpy(), r.inv.cpu().numpy(), r.flags.cpu().numpy()


def bits_corpus(n, rng):
    bits = rng.integers(0, 2 ** 63, size=(n, 9), dtype=np.int64) * rng.choice([1, -1], size=(n, 9))
    a = bits.view(np.float64).copy()
    pick = rng.random((n, 9)) < rng.uniform(0.3, 0.95)
    return np.ascontiguousarray(np.where(pick, rng.standard_normal((n, 9)), a))


def main():
    batches = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    n = 1 << (int(sys.argv[2]) if len(sys.argv) > 2 else 22)
    first = int(sys.argv[3]) if len(sys.argv) > 3 else 0
    t0 = time.time()
    checked = 0
    for b in range(first, first + batches):
        rng = np.random.default_rng(1000 + b)
        corpora = {
            "bits": bits_corpus(n, rng),
            "mixed": U.mixed_corpus(n, 2000 + b),
            "edges": _moderate_edge_corpus(n, 3000 + b),
        }
        for cfg in (1, 2, 3, 4, 5):
            corpora[f"config{cfg}"] = eig.generate(cfg, n, seed=4000 + 10 * b + cfg).cpu().numpy()
        for name, a in corpora.items():
            lam, inv, flags = run(a)
            _assert_parity(a, lam, inv, flags, f"batch {b} {name}",
                           lam_tol_fallback=_exact.within_reference_forward_error if name == "config4" else None)
            # invariants-only entry point: same bits as the fused kernel's
            inv2 = eig.invariants(torch.from_numpy(a).cuda()).cpu().numpy()
            assert U.bit_equal(inv2, inv).all(), f"batch {b} {name}: invariants entry differs"
            # eigvalss on the mirrored corpus: equals eigvals bit for bit, no rejects
            s_ = a.copy()
            s_[:, [3, 6, 7]] = s_[:, [1, 2, 5]]
            rs = eig.eigvalss(torch.from_numpy(s_).cuda(), return_flags=True)
            re = eig.eigvals(torch.from_numpy(s_).cuda())
            fl = rs.flags.cpu().numpy()
            ok = (fl & 2) == 0  # NaN/inf records may still fail the gate, as in the reference
            assert U.bit_equal(rs.lam.cpu().numpy()[ok], re.lam.cpu().numpy()[ok]).all(), \
                f"batch {b} {name}: eigvalss != eigvals on symmetric input"
            checked += a.shape[0]
        print(f"batch {b}: {len(corpora)} corpora x {n} records ok ({time.time() - t0:.0f} s)", flush=True)
    print(f"fuzz ok: {checked} records")


if __name__ == "__main__":
    main()
