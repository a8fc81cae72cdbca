"""GPU parity: the sm_100a kernels, called through the C ABI, against the
checker (compiled reference core when present, else the C restatement), run
on this box's host cores in the same process (lambda bits depend on the host
libm -- SURVEY 0.6).

Gates (BASELINE north_star): invariants bit-exact (NaN == NaN), advisory and
NotSymmetric flags bit-exact, lambda within 4 * 2^-52 * max|lambda_ref|
(TOL_UNITS) with identical non-finite classes; config 4 (ill-conditioned
eigenbasis) falls back to the reference's own forward error where the 4-ulp
test fails (tests/_exact.py).
"""
import ctypes
import os
import subprocess

import numpy as np
import pytest

from tests import _util as U

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2511_00292_b200 as eig  # noqa: E402

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "eig33_golden.npz")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.fail("gpu tests need a CUDA device")  # loud: no silent CPU pass
    eig.lib()
    yield
    torch.cuda.synchronize()


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64).reshape(-1, 9)).cuda()


def _run(a_host, *, inv=True, flags=True):
    r = eig.eigvals(_dev(a_host), return_invariants=inv, return_flags=flags)
    torch.cuda.synchronize()
    return [None if x is None else x.cpu().numpy() for x in r]


def _assert_parity(a, lam, inv, flags, name, max_units=None, lam_tol_fallback=None):
    """Invariants and flags bitwise; lambda through U.lam_gate (strict reading,
    4 ulp(max|lam_ref|), libm-misrounding exceptions inside the loose reading)."""
    inv_r = U.checker_invariants(a)
    bad = ~U.bit_equal(inv, inv_r).all(axis=1)
    assert not bad.any(), f"{name}: {bad.sum()} invariant rows differ, first {np.nonzero(bad)[0][:5]}"
    lam_r, adv_r = U.checker_eigvals(a)
    if flags is not None:
        fb = (flags & eig.FLAG_ADVISORY) != adv_r
        assert not fb.any(), f"{name}: advisory differs on {fb.sum()} records"
    es, el, explained = U.lam_gate(a, lam, lam_r, inv_ref=inv_r, fallback=lam_tol_fallback)
    if max_units is not None:
        assert el.max() <= max_units, f"{name}: worst {el.max():.3g} units"
    return el


def test_golden_fixtures_on_device():
    g = np.load(GOLDEN)
    lam, inv, flags = _run(g["a"])
    assert U.bit_equal(inv, g["inv"]).all()
    assert ((flags & 1) == g["adv"]).all()
    U.lam_gate(g["a"], lam, g["lam"])
    _assert_parity(g["a"], lam, inv, flags, "golden")


def test_known_answers_on_device():
    a = np.array([U.KAT_MATRICES[k] for k in ("diag(-1,1,2)", "diag(1,2,3)", "rotation", "7.25*I")]
                 + [U.perf_matrix()], dtype=np.float64)
    lam, inv, flags = _run(a)
    assert inv[0][3] == 36.0 and inv[0][0] == 2.0
    assert inv[1][1] == 1.0 and inv[1][2] == 0.0
    assert inv[2][3] == -16.0 and flags[2] & 1 and np.isfinite(lam[2]).all()
    assert (lam[3] == 7.25).all()
    assert np.abs(lam[1] - [1, 2, 3]).max() <= 1e-14
    assert [np.float64(x).view(np.uint64) for x in inv[4]] == [
        0x3FF000000000002C, 0x3FF5555555555573, 0xBFE2F684BDA12F8F, 0x3A5F620000000030]


def test_triple_angle_kats():
    ta = np.load(GOLDEN)
    j3 = torch.tensor(ta["ta_in"][:, 0], dtype=torch.float64, device="cuda")
    dc = torch.tensor(ta["ta_in"][:, 1], dtype=torch.float64, device="cuda")
    phi = eig.triple_angle(j3, dc).cpu().numpy()
    assert U.bit_equal(phi, ta["ta"]).all()
    assert phi[0] == np.pi / 2 and phi[1] == 0.0 and phi[2] == np.pi and phi[3] == 0.0


@pytest.mark.parametrize("config,n", [(1, 1 << 20), (2, 1 << 22), (3, 1 << 22), (4, 1 << 22),
                                      (5, 1 << 22)])
def test_config_parity_full_size(config, n):
    """BASELINE configs at their full batch (config 3 at 2^22 of its 2^28; the
    full 2^28 is covered by test_config3_full_properties)."""
    a_d = eig.generate(config, n, seed=1000 + config)
    r = eig.eigvals(a_d, return_invariants=True, return_flags=True)
    torch.cuda.synchronize()
    a = a_d.cpu().numpy()
    lam, inv, flags = (x.cpu().numpy() for x in r)
    fallback = None
    if config == 4:
        from tests import _exact
        fallback = _exact.within_reference_forward_error
    err = _assert_parity(a, lam, inv, flags, f"config{config}", lam_tol_fallback=fallback)
    assert (err == 0).mean() > 0.99  # most records reproduce the reference bits exactly


def test_config3_full_size_every_record():
    """Config 3 at its full 2^28 batch (19.3 GB in): every record against the
    compiled reference on this box's host cores -- invariants bit-exact,
    lambda within tolerance -- plus the size-independent properties of
    proj/tests/test_eigensolver.cpp:83-102 (ascending order, trace consistency)
    evaluated on the device for every record."""
    n = 1 << 28
    free, _ = torch.cuda.mem_get_info()
    if free < n * (72 + 24 + 32 + 8) + (4 << 30):
        pytest.skip("not enough device memory for the 2^28 batch")
    try:
        import psutil
        if psutil.virtual_memory().available < 80e9:
            pytest.skip("not enough host memory for the full-size reference comparison")
    except ImportError:
        pass
    a_d = eig.generate(3, n, seed=3)
    r = eig.eigvals(a_d, return_invariants=True)
    lam, inv = r.lam, r.inv
    l1, l2, l3 = lam[:, 0], lam[:, 1], lam[:, 2]
    assert bool(((l1 <= l2) & (l2 <= l3)).all())
    a9 = a_d.view(n, 9)
    i1 = (a9[:, 0] + a9[:, 4]) + a9[:, 8]
    s = (l1 + l2) + l3
    spread = 2.0 * torch.sqrt(3.0 * torch.clamp(inv[:, 1], min=0.0))
    assert bool(((s - i1).abs() <= 20 * 2.0 ** -53 * (i1.abs() + spread)).all())
    del s, spread, i1, l1, l2, l3
    a = a_d.cpu().numpy()
    del a_d
    lam_h = lam.cpu().numpy()
    inv_h = inv.cpu().numpy()
    del lam, inv, r
    step = 1 << 25  # compare in slices to bound host temporaries
    worst = worst_strict = 0.0
    exact = 0
    explained = 0
    for lo in range(0, n, step):
        sl = slice(lo, lo + step)
        inv_r = U.checker_invariants(a[sl])
        assert U.bit_equal(inv_h[sl], inv_r).all(), f"invariants differ in [{lo}, {lo + step})"
        lam_r, _ = U.checker_eigvals(a[sl], adv=False)
        es, el, ex = U.lam_gate(a[sl], lam_h[sl], lam_r, inv_ref=inv_r)
        worst = max(worst, float(el.max()))
        worst_strict = max(worst_strict, float(es.max()))
        explained += len(ex)
        exact += int((el == 0).sum())
    assert worst <= U.TOL_UNITS, worst
    assert explained <= 64, explained
    assert exact / n > 0.998


def test_mixed_corpus_and_nonfinite_classes():
    a = U.mixed_corpus(1 << 20, 17)
    lam, inv, flags = _run(a)
    _assert_parity(a, lam, inv, flags, "mixed")


def test_moderate_range_edges():
    """Records at both ends of the moderate tier's range [2^-100, 2^100) (finest
    grains, near-scalar records with off-diagonals down to 2^-97, grid records
    scaled to 2^+-90) take the guard-free tiers and reproduce the reference."""
    from tests.test_hostmath import _moderate_edge_corpus

    a = _moderate_edge_corpus(1 << 20, 53)
    lam, inv, flags = _run(a)
    _assert_parity(a, lam, inv, flags, "moderate edges")


@pytest.mark.parametrize("n", [1, 2, 3, 255, 256, 257, 511, 4097, 100003])
def test_ragged_sizes_and_tails(n):
    a = U.mixed_corpus(max(n, 8), n)[:n]
    lam, inv, flags = _run(a)
    _assert_parity(a, lam, inv, flags, f"n={n}")


def test_empty_batch():
    r = eig.eigvals(torch.empty((0, 9), dtype=torch.float64, device="cuda"), return_invariants=True)
    assert r.lam.shape == (0, 3) and r.inv.shape == (0, 4)


def test_misaligned_input_uses_coalesced_path():
    n = 70001
    a = U.mixed_corpus(n, 5)
    buf = torch.empty(n * 9 + 1, dtype=torch.float64, device="cuda")
    buf[1:] = torch.from_numpy(a.reshape(-1)).cuda()
    view = buf[1:].view(n, 9)  # 8-B aligned, not 16-B: no TMA
    assert view.data_ptr() % 16 == 8
    r = eig.eigvals(view, return_invariants=True, return_flags=True)
    torch.cuda.synchronize()
    _assert_parity(a, r.lam.cpu().numpy(), r.inv.cpu().numpy(), r.flags.cpu().numpy(), "misaligned")


def test_unaligned_invariants_output_equals_aligned():
    """Invariant outputs that are not 32-B aligned take four 8-B stores instead
    of one 256-bit store: same bits, both entry points, ragged sizes."""
    L = eig.lib()
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    P = lambda t: ctypes.c_void_p(t.data_ptr())
    for n in (1, 31, 4099, (1 << 20) + 3):
        a_d = eig.generate(5, n, seed=n)
        lam = torch.empty((n, 3), dtype=torch.float64, device="cuda")
        fl = torch.empty(n, dtype=torch.uint8, device="cuda")
        ref = eig.eigvals(a_d, return_invariants=True).inv
        for off in (8, 16, 24):
            buf = torch.zeros(n * 4 + 4, dtype=torch.float64, device="cuda")
            p = ctypes.c_void_p(buf.data_ptr() + off)
            assert L.eig33cu_eigvals(P(a_d), n, p, P(lam), P(fl), st) == 0
            got = buf[off // 8: off // 8 + 4 * n].view(n, 4)
            torch.cuda.synchronize()
            assert U.bit_equal(got.cpu().numpy(), ref.cpu().numpy()).all(), (n, off)
            buf.zero_()
            assert L.eig33cu_invariants(P(a_d), n, p, st) == 0
            torch.cuda.synchronize()
            assert U.bit_equal(got.cpu().numpy(), ref.cpu().numpy()).all(), (n, off, "invariants")


def test_invariants_only_entry_point():
    a_d = eig.generate(5, 1 << 21, seed=9)
    inv = eig.invariants(a_d).cpu().numpy()
    assert U.bit_equal(inv, U.checker_invariants(a_d.cpu().numpy())).all()


def test_eigvalss_device_and_host():
    a_d = eig.generate(1, 1 << 20, seed=77)  # bitwise symmetric
    r_s = eig.eigvalss(a_d, return_invariants=True, return_flags=True)
    r_g = eig.eigvals(a_d, return_invariants=True)
    torch.cuda.synchronize()
    assert U.bit_equal(r_s.lam.cpu().numpy(), r_g.lam.cpu().numpy()).all()
    assert (r_s.flags.cpu().numpy() == 0).all()
    lam_r, st_r = U.checker_eigvalss(a_d.cpu().numpy())
    assert (st_r == 0).all()
    U.lam_gate(a_d.cpu().numpy(), r_s.lam.cpu().numpy(), lam_r)
    # symmetry gate (test_eigensolver.cpp:150-165) -> flag bit1 on device, ValueError on host
    bad = np.array([[1.0, 1.0, 0, 1.0 + 1e-8, 2, 0, 0, 0, 3], U.KAT_MATRICES["rotation"],
                    [1.0, 1.0, 0, 1.0 + 2.0 ** -52, 2, 0, 0, 0, 3]])
    r = eig.eigvalss(_dev(bad), return_flags=True)
    f = r.flags.cpu().numpy()
    assert list((f & eig.FLAG_NOT_SYMMETRIC) != 0) == [True, True, False]
    with pytest.raises(ValueError):
        eig.eigvalss(bad)
    lam_h = eig.eigvalss(bad[2:]).lam
    lam_c, _ = U.checker_eigvalss(bad[2:])
    U.lam_gate(bad[2:], lam_h, lam_c)


def test_host_entry_points_equal_device_entry_points():
    a_d = eig.generate(3, (1 << 22) + 5, seed=42)
    r_d = eig.eigvals(a_d, return_invariants=True, return_flags=True)
    a = a_d.cpu().numpy()
    r_h = eig.eigvals(a, return_invariants=True, return_flags=True)
    assert U.bit_equal(r_h.lam, r_d.lam.cpu().numpy()).all()
    assert U.bit_equal(r_h.inv, r_d.inv.cpu().numpy()).all()
    assert (r_h.flags == r_d.flags.cpu().numpy()).all()
    r_m = eig.multi_eigvals(a, 1, return_invariants=True)
    assert U.bit_equal(r_m.lam, r_h.lam).all()
    assert U.bit_equal(eig.invariants(a), r_h.inv).all()


def test_host_pipeline_reuses_staging_sets():
    """Host-buffer API over more chunks than staging sets (7 x 2^22 + 3 records,
    3 sets): every chunk's kernel must see its own H2D copy, never a stale
    buffer, with the kernels launched under programmatic dependent launch."""
    n = 7 * (1 << 22) + 3
    a_d = eig.generate(3, n, seed=77)
    want = eig.eigvals(a_d).lam.cpu().numpy()
    a = a_d.cpu().numpy()
    del a_d
    for _ in range(2):
        got = eig.eigvals(a).lam
        assert U.bit_equal(got, want).all()


def test_host_staged_path_all_outputs():
    """Pageable host batches >= 8 MB take the pinned-bounce staged pipeline:
    every output (lambda, invariants, flags; eigvalss rejects; invariants-only)
    equals the device path, including a ragged last chunk."""
    n = 3 * (1 << 20) + 333
    a_d = eig.generate(4, n, seed=88)
    a = a_d.cpu().numpy()
    r_d = eig.eigvals(a_d, return_invariants=True, return_flags=True)
    r_h = eig.eigvals(a, return_invariants=True, return_flags=True)
    assert U.bit_equal(r_h.lam, r_d.lam.cpu().numpy()).all()
    assert U.bit_equal(r_h.inv, r_d.inv.cpu().numpy()).all()
    assert (r_h.flags == r_d.flags.cpu().numpy()).all()
    assert U.bit_equal(eig.invariants(a), r_d.inv.cpu().numpy()).all()
    s_ = a.copy()
    s_[:, [3, 6, 7]] = s_[:, [1, 2, 5]]
    rs_h = eig.eigvalss(s_, return_flags=True)
    rs_d = eig.eigvalss(torch.from_numpy(s_).cuda(), return_flags=True)
    assert U.bit_equal(rs_h.lam, rs_d.lam.cpu().numpy()).all()
    s_[n - 2, 1] += 1.0  # one asymmetric record in the last chunk
    with pytest.raises(ValueError):
        eig.eigvalss(s_)


def _device_lists():
    ng = torch.cuda.device_count() if torch.cuda.is_available() else 1
    lists = [[0], [0, 0], [0, 0, 0, 0, 0]]  # repeated devices: threads take turns on one pipeline
    if ng >= 2:
        lists += [list(range(ng)), [ng - 1, 0]]
    return lists


@pytest.mark.parametrize("devices", _device_lists())
def test_multi_gpu_entry_points_on_available_devices(devices):
    """eig33_multi_eigvals_on over shard->device lists give the single-device
    bits (pageable input large enough for the staged pipeline, so the shard
    threads' host copies run concurrently through the shared copy pool); the
    ngpu form over every visible device too; asking for more devices than
    exist is an error."""
    ng = torch.cuda.device_count()
    if ng < 2:
        print(f"NOTE: only {ng} CUDA device visible -- shards run on repeated device lists; "
              "the cross-device path needs a multi-GPU box")
    a = U.mixed_corpus(len(devices) * (1 << 18) + 11, 61)  # >= 8 MB pageable per shard
    r1 = eig.eigvals(a, return_invariants=True, return_flags=True)
    rm = eig.multi_eigvals(a, devices=devices, return_invariants=True, return_flags=True)
    assert U.bit_equal(rm.lam, r1.lam).all() and U.bit_equal(rm.inv, r1.inv).all()
    assert (rm.flags == r1.flags).all()
    rn = eig.multi_eigvals(a, ng, return_invariants=True, return_flags=True)
    assert U.bit_equal(rn.lam, r1.lam).all() and (rn.flags == r1.flags).all()
    assert U.bit_equal(eig.multi_invariants(a, ng), r1.inv).all()
    s_ = a.copy()
    s_[:, [3, 6, 7]] = s_[:, [1, 2, 5]]
    assert U.bit_equal(eig.multi_eigvalss(s_, ng).lam, eig.eigvalss(s_).lam).all()
    with pytest.raises(ValueError):
        eig.multi_eigvals(a, ng + 1)
    with pytest.raises(ValueError):
        eig.multi_eigvals(a, devices=[0, ng])


def test_not_symmetric_reports_first_record():
    """The batched eigvalss names the first record failing the gate -- the one
    a loop of scalar calls throws on (src/eigensolver.cpp:102) -- through the C
    ABI (eig33cu_last_notsym_index), the error text and the multi-GPU driver."""
    a = eig.generate(1, (1 << 20) + 3, seed=5).cpu().numpy()  # bitwise symmetric, pageable
    L = eig.lib()
    for k in (0, 77, (1 << 19) + 1, (1 << 20) + 2):
        b = a.copy()
        b[k, 1] += 0.25
        b[min(k + 5, b.shape[0] - 1), 5] += 0.25  # a second, later offender
        first = k
        with pytest.raises(ValueError, match=f"record {first}"):
            eig.eigvalss(b)
        assert L.eig33cu_last_notsym_index() == first
        with pytest.raises(ValueError, match=f"record {first}"):
            eig.multi_eigvalss(b, 1)
        assert L.eig33cu_last_notsym_index() == first
    eig.eigvalss(a)
    assert L.eig33cu_last_notsym_index() == -1


def test_host_call_restores_current_device():
    """eig33_*_host switch to the requested device and restore the caller's
    current device on return (a rank that did set_device(k) keeps k)."""
    ng = torch.cuda.device_count()
    a = U.mixed_corpus(1000, 3)
    for cur in range(ng):
        torch.cuda.set_device(cur)
        for target in range(ng):
            eig.eigvals(a, device=target)
            assert torch.cuda.current_device() == cur
    torch.cuda.set_device(0)


def test_error_return_leaves_no_pending_copies():
    """A failing host call (device index out of range mid-batch for the
    multi-driver) returns an error and leaves the library usable."""
    a = U.mixed_corpus(1 << 18, 4)
    with pytest.raises(ValueError):
        eig.eigvals(a, device=torch.cuda.device_count())
    r = eig.eigvals(a)
    assert np.isfinite(r.lam[: 1 << 16]).any()


def test_shard_invariance_bitwise():
    """Results are identical whatever the contiguous even-aligned sharding
    (the multi-GPU driver's partition), emulated on one device."""
    n = 3_000_001
    a_d = eig.generate(5, n, seed=5)
    full = eig.eigvals(a_d, return_invariants=True).lam
    for g in (2, 4, 8):
        bounds = [2 * (k * n // (2 * g)) for k in range(g)] + [n]
        parts = [eig.eigvals(a_d[lo:hi]).lam for lo, hi in zip(bounds[:-1], bounds[1:])]
        assert torch.equal(torch.cat(parts).view(torch.int64), full.view(torch.int64))


@pytest.mark.parametrize("config", [1, 2, 3, 4, 5])
def test_device_generator_equals_host_regeneration(config):
    """eig33cu_generate and the host regeneration (oracle/libcorpus.so, used by
    bench.py's reference arm) share eig33_gen_core.h and must agree bitwise --
    the reference arm times the reference on exactly the GPU arm's records."""
    for seed, first, n in ((1000 + config, 0, 1 << 16), (0x251100292, (1 << 20) - 3000, 1 << 13),
                           (7, (3 << 20) - 77, 1 << 12), (2 ** 64 - 1, 12345678901, 999)):
        dev = eig.generate(config, n, seed=seed, first_index=first).cpu().numpy()
        host = U.host_corpus(config, n, seed, first)
        same = dev.view(np.uint64) == host.view(np.uint64)
        assert same.all(), f"config {config} seed {seed} first {first}: {(~same.all(axis=1)).sum()} records differ"


def test_generator_is_counter_based():
    a = eig.generate(3, 1 << 16, seed=11)
    b = eig.generate(3, 1 << 15, seed=11, first_index=1 << 15)
    assert torch.equal(a[1 << 15:], b)
    c1 = eig.generate(1, 4096, seed=1).cpu().numpy()
    assert (c1[:, [3, 6, 7]] == c1[:, [1, 2, 5]]).all()  # bitwise symmetric


def test_cxx_batch_api_links_and_runs(tmp_path):
    exe = tmp_path / "batch_api_check"
    src = os.path.join(U.ROOT, "tests", "cpp", "batch_api_check.cpp")
    so_dir = os.path.join(U.ROOT, "paper_2511_00292_b200")
    r = subprocess.run(["g++", "-std=c++17", "-DEIG33_STANDALONE_TYPES", "-I",
                        os.path.join(U.ROOT, "include"), src, "-o", str(exe),
                        os.path.join(so_dir, "_eig33cuda.so"), "-Wl,-rpath," + so_dir],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0 and out.stdout.strip() == "OK", out.stdout + out.stderr


def test_cxx_batch_api_over_reference_types_runs():
    """The same consumer compiled against the REFERENCE's own headers (its Mat3,
    InvariantSet, EigenTriple and NotSymmetric; built by build() where
    /root/reference exists, shipped prebuilt) links with the product library and
    runs on the GPU: the drop-in overloads over the reference's real types."""
    from paper_2511_00292_b200 import build

    exe = build.REF_CXX_CHECK
    assert os.path.exists(exe), f"{exe} missing: run __graft_entry__.build() where /root/reference exists"
    out = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0 and out.stdout.strip() == "OK", out.stdout + out.stderr


def test_variant_invariants_host_entry_equals_device():
    """eig33_invariants_variant_host (pageable direct, pageable staged) gives
    the device entry's bits for all three variants."""
    for n in (1000, (1 << 17) + 3):
        a = U.mixed_corpus(n, 29)
        d = torch.from_numpy(a).cuda()
        for v in ("Stable", "Naive", "NaiveTensor"):
            assert U.bit_equal(eig.invariants(a, variant=v), eig.invariants(d, variant=v).cpu().numpy()).all()


@pytest.mark.parametrize("n,offset", [((1 << 18), 0), (4099, 0), (1, 0), (70001, 1)])
def test_study_variants_on_device(n, offset):
    """naive / tensor invariants, eigvals_naive (+advisory), Jacobians vs the
    compiled reference: bit-exact except eigvals_naive's lambda (tolerance).
    The study kernels run on the hot path's TMA ring and chunk scheduler; a
    ragged size and a record base that is only 8-B aligned (offset 1: the
    cooperative-load path) are covered too."""
    base = U.mixed_corpus(n + 1, 31 + n)
    a = base[offset:offset + n]
    R = U.ref()
    if offset:  # device input at an 8-B aligned (not 16-B aligned) address
        buf = torch.from_numpy(np.ascontiguousarray(base).reshape(-1)).cuda()
        a_dev = buf[9 * offset: 9 * (offset + n)].view(n, 9)
        assert a_dev.data_ptr() % 16 != 0
        inv_d = eig.invariants(a_dev, variant="Naive").cpu().numpy()
        want = np.empty((n, 4))
        R.ref_invariants_variant(U.ptr(np.ascontiguousarray(a)), U.S(n), 1, U.ptr(want), U.nthreads())
        assert U.bit_equal(inv_d, want).all()
    a = np.ascontiguousarray(a)
    for name, v in (("Naive", 1), ("NaiveTensor", 2)):
        got = eig.invariants(a, variant=name)
        want = np.empty((n, 4))
        R.ref_invariants_variant(U.ptr(a), U.S(n), v, U.ptr(want), U.nthreads())
        assert U.bit_equal(got, want).all(), name
    r = eig.eigvals_naive(a, return_flags=True)
    lam, fl = np.empty((n, 3)), np.empty(n, np.uint8)
    R.ref_eigvals_naive(U.ptr(a), U.S(n), U.ptr(lam), U.ptr(fl), U.nthreads())
    assert ((r.flags & 1) == fl).all()
    assert (U.lam_error_units(r.lam, lam) <= U.TOL_UNITS).all()
    j2, j3, jd = eig.jacobians(a)
    want = [np.empty((n, 9)) for _ in range(3)]
    R.ref_jacobians(U.ptr(a), U.S(n), *(U.ptr(w) for w in want), U.nthreads())
    for got, w in zip((j2, j3, jd), want):
        assert U.bit_equal(got.reshape(n, 9), w).all()


# ---- properties the reference's own tests assert, re-run on GPU outputs ----

def _mm(x, y):
    """Reference matmul association (src/mat3.cpp:18-26), batched."""
    return ((x[:, :, 0, None] * y[:, None, 0, :] + x[:, :, 1, None] * y[:, None, 1, :])
            + x[:, :, 2, None] * y[:, None, 2, :])


def _inv_adj(v):
    """Reference inverse_adjugate (src/mat3.cpp:49-64), batched."""
    c = np.empty_like(v)
    c[:, 0, 0] = v[:, 1, 1] * v[:, 2, 2] - v[:, 1, 2] * v[:, 2, 1]
    c[:, 0, 1] = v[:, 1, 2] * v[:, 2, 0] - v[:, 1, 0] * v[:, 2, 2]
    c[:, 0, 2] = v[:, 1, 0] * v[:, 2, 1] - v[:, 1, 1] * v[:, 2, 0]
    c[:, 1, 0] = v[:, 0, 2] * v[:, 2, 1] - v[:, 0, 1] * v[:, 2, 2]
    c[:, 1, 1] = v[:, 0, 0] * v[:, 2, 2] - v[:, 0, 2] * v[:, 2, 0]
    c[:, 1, 2] = v[:, 0, 1] * v[:, 2, 0] - v[:, 0, 0] * v[:, 2, 1]
    c[:, 2, 0] = v[:, 0, 1] * v[:, 1, 2] - v[:, 0, 2] * v[:, 1, 1]
    c[:, 2, 1] = v[:, 0, 2] * v[:, 1, 0] - v[:, 0, 0] * v[:, 1, 2]
    c[:, 2, 2] = v[:, 0, 0] * v[:, 1, 1] - v[:, 0, 1] * v[:, 1, 0]
    det = (v[:, 0, 0] * (v[:, 1, 1] * v[:, 2, 2] - v[:, 1, 2] * v[:, 2, 1])
           - v[:, 0, 1] * (v[:, 1, 0] * v[:, 2, 2] - v[:, 1, 2] * v[:, 2, 0])) \
        + v[:, 0, 2] * (v[:, 1, 0] * v[:, 2, 1] - v[:, 1, 1] * v[:, 2, 0])
    return np.transpose(c, (0, 2, 1)) / det[:, None, None], det


def test_acceptance_c9_ordering_and_trace_on_1e6_spectra():
    """proj/tests/acceptance/acceptance.cpp:244-265 (C9): ascending order and
    trace consistency on 10^6 random similarity transforms."""
    rng = np.random.default_rng(9)
    n = 1_000_000
    m = rng.uniform(-1, 1, (int(n * 1.2), 3, 3))
    minv, det = _inv_adj(m)
    keep = np.abs(det) >= 1e-2
    m, minv = m[keep][:n], minv[keep][:n]
    d = rng.uniform(-5, 5, (n, 3))
    a = _mm(m * d[:, None, :], minv).reshape(n, 9)
    lam, inv, _ = _run(a, flags=False)
    assert ((lam[:, 0] <= lam[:, 1]) & (lam[:, 1] <= lam[:, 2])).all()
    i1 = inv[:, 0]
    spread = 2.0 * np.sqrt(3.0 * np.maximum(inv[:, 1], 0.0))
    s = (lam[:, 0] + lam[:, 1]) + lam[:, 2]
    assert (np.abs(s - i1) <= 20 * 2.0 ** -53 * (np.abs(i1) + spread)).all()


def test_scaled_identities_exact():
    """test_eigensolver.cpp:41-52 and acceptance C2: lambda == alpha bitwise,
    j2 = j3 = disc = 0, no advisory, for alpha = mant*2^[-30,30] and 10^U[-100,100]."""
    rng = np.random.default_rng(2)
    al = np.concatenate([np.ldexp(rng.uniform(-1, 1, 5000), rng.integers(-30, 31, 5000)),
                         10.0 ** rng.uniform(-100, 100, 5000)])
    a = np.zeros((al.size, 9))
    a[:, 0] = a[:, 4] = a[:, 8] = al
    lam, inv, flags = _run(a)
    assert (lam == al[:, None]).all() and (inv[:, 1:] == 0).all() and not (flags & 1).any()


def test_symmetric_disc_is_nonnegative():
    """test_invariants.cpp:169-182 (500 matrices, U(-5,5), seed 23) at 2^20 records:
    disc_stable of a bitwise-symmetric matrix is a sum of squares, so >= 0, and
    no symmetric record raises the advisory; eigvalss equals eigvals there."""
    rng = np.random.default_rng(23)
    n = 1 << 20
    a = rng.uniform(-5, 5, (n, 9))
    a[:, [3, 6, 7]] = a[:, [1, 2, 5]]
    lam, inv, flags = _run(a)
    _assert_parity(a, lam, inv, flags, "symmetric U(-5,5)")
    assert (inv[:, 3] >= 0.0).all()
    assert not (flags & 1).any()
    rs = eig.eigvalss(_dev(a), return_flags=True)
    assert U.bit_equal(rs.lam.cpu().numpy(), lam).all()
    assert not (rs.flags.cpu().numpy() & 2).any()


def test_shift_equivariance():
    """test_eigensolver.cpp:104-128: entries and shifts on a 2^-20 grid, worst
    |(l(A)+beta) - l(A+beta I)| / (eps*(|beta| + ||A||_F)) <= 30."""
    rng = np.random.default_rng(33)
    n = 200_000
    snap = lambda x: np.ldexp(np.round(np.ldexp(x, 20)), -20)
    a = snap(rng.uniform(-4, 4, (n, 9)))
    beta = snap(rng.uniform(-4, 4, n))
    sh = a.copy()
    sh[:, [0, 4, 8]] += beta[:, None]
    l0, _, _ = _run(a, inv=False, flags=False)
    l1, _, _ = _run(sh, inv=False, flags=False)
    scale = 2.0 ** -53 * (np.abs(beta) + np.sqrt((a * a).sum(1)))
    diff = np.abs((l0 + beta[:, None]) - l1).max(1)
    assert (diff / scale).max() <= 30.0


def test_eigvalss_tight_symmetric_cluster():
    """test_eigensolver.cpp:140-146: spectrum error <= 10 eps ||A||_F on
    U diag(1,1,1+1e-12) U^T (Symm transform, bench.cpp:53-60)."""
    q = np.sqrt(2.0) / 2.0
    u = np.array([[q, -0.5, 0.5], [q, 0.5, -0.5], [0.0, q, q]])
    d = np.diag([1.0, 1.0, 1.0 + 1e-12])
    a = _mm(_mm(u[None], d[None]), u.T[None]).reshape(1, 9)
    lam = eig.eigvalss(a).lam[0]
    assert np.abs(lam - [1.0, 1.0, 1.0 + 1e-12]).max() <= 10 * 2.0 ** -53 * np.sqrt((a * a).sum())


def test_signed_zeros_and_sparse_records():
    """Exact +-0 entries go through the moderate tiers (a zero is a multiple of
    every grain); signs of zero must survive into j3/disc and the triple angle
    (atan2(+0, -0) = pi) exactly as in the reference."""
    rng = np.random.default_rng(71)
    n = 1 << 18
    a = np.round(rng.standard_normal((n, 9)) * 8) / 8
    z = rng.random((n, 9)) < 0.4
    a[z] = np.where(rng.random(z.sum()) < 0.5, 0.0, -0.0)
    a[: n // 16] = np.where(rng.random((n // 16, 9)) < 0.5, 0.0, -0.0)  # all-zero records
    lam, inv, flags = _run(a)
    _assert_parity(a, lam, inv, flags, "signed-zeros")


def test_concurrent_host_threads_and_streams():
    """The C ABI is reentrant: host threads calling the host-buffer API and
    device calls on independent streams give the single-call bits."""
    import threading

    a = U.mixed_corpus(1 << 18, 81)
    want = eig.eigvals(a, return_invariants=True)
    res = [None] * 4

    def work(i):
        res[i] = eig.eigvals(a, return_invariants=True)

    th = [threading.Thread(target=work, args=(i,)) for i in range(4)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for r in res:
        assert U.bit_equal(r.lam, want.lam).all() and U.bit_equal(r.inv, want.inv).all()
    d = _dev(a)
    streams = [torch.cuda.Stream() for _ in range(3)]
    outs = []
    for s in streams:
        with torch.cuda.stream(s):
            outs.append(eig.eigvals(d).lam)
    torch.cuda.synchronize()
    for o in outs:
        assert U.bit_equal(o.cpu().numpy(), want.lam).all()


def test_dependent_launches_in_stream_order():
    """k_fused / k_invariants start under programmatic dependent launch: their
    prologue may overlap the previous kernel, but no caller buffer is touched
    before griddepcontrol.wait.  Chain kernels where each one reads (RAW) or
    overwrites (WAR) what the previous one wrote, with no host sync in between,
    and compare with the same chain run one synchronised call at a time."""
    n = 3 * (1 << 18)  # lam of n records = n/3 records of 9 doubles
    a = eig.generate(3, n, seed=404)
    L = eig.lib()
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    P = lambda t: ctypes.c_void_p(t.data_ptr())

    def chain(sync):
        lam = torch.empty((n, 3), dtype=torch.float64, device="cuda")
        inv = torch.empty((n // 3, 4), dtype=torch.float64, device="cuda")
        lam2 = torch.empty((n // 3, 3), dtype=torch.float64, device="cuda")
        outs = []
        for rep in range(3):
            assert L.eig33cu_eigvals(P(a), n, None, P(lam), None, st) == 0          # writes lam
            if sync:
                torch.cuda.synchronize()
            assert L.eig33cu_invariants(P(lam), n // 3, P(inv), st) == 0            # RAW on lam
            if sync:
                torch.cuda.synchronize()
            assert L.eig33cu_eigvals(P(lam), n // 3, None, P(lam2), None, st) == 0  # RAW on lam
            if sync:
                torch.cuda.synchronize()
            lam.fill_(float(rep))                                                   # WAR on lam
            outs += [inv.clone(), lam2.clone()]
        torch.cuda.synchronize()
        return [o.cpu().numpy() for o in outs]

    want = chain(True)
    for _ in range(3):
        got = chain(False)
        for g, w in zip(got, want):
            assert U.bit_equal(g, w).all()


def test_cuda_graph_capture_and_replay():
    """The device entry points can be captured in a CUDA graph (the fused
    kernels' programmatic-launch edges included) and replayed: same bits as
    eager calls, and replays see new input contents."""
    n = (1 << 18) + 37
    a = eig.generate(4, n, seed=515)
    L = eig.lib()
    P = lambda t: ctypes.c_void_p(t.data_ptr())
    lam = torch.empty((n, 3), dtype=torch.float64, device="cuda")
    inv = torch.empty((n, 4), dtype=torch.float64, device="cuda")
    fl = torch.empty((n,), dtype=torch.uint8, device="cuda")
    lam2 = torch.empty((n // 3, 3), dtype=torch.float64, device="cuda")

    def calls(st):
        assert L.eig33cu_eigvals(P(a), n, P(inv), P(lam), P(fl), st) == 0
        assert L.eig33cu_eigvals(P(lam), n // 3, None, P(lam2), None, st) == 0  # reads lam (RAW)

    calls(ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))  # eager warm-up
    torch.cuda.synchronize()
    want = [x.clone() for x in (lam, inv, fl, lam2)]
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for x in (lam, inv, fl, lam2):
            x.zero_()
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            calls(ctypes.c_void_p(s.cuda_stream))
    g.replay()
    torch.cuda.synchronize()
    for x, w in zip((lam, inv, fl, lam2), want):
        assert torch.equal(x.view(torch.uint8), w.view(torch.uint8))
    b = eig.generate(5, n, seed=516)
    a.copy_(b)  # new contents, same buffer: the replay must pick them up
    g.replay()
    torch.cuda.synchronize()
    r = eig.eigvals(b, return_invariants=True, return_flags=True)
    assert torch.equal(lam.view(torch.uint8), r.lam.view(torch.uint8))
    assert torch.equal(inv.view(torch.uint8), r.inv.view(torch.uint8))
    assert torch.equal(fl, r.flags)


def test_generate_case_matches_reference_bitwise():
    """Batched paper corpora (src/bench.cpp:53-82) on the device equal the
    compiled reference's own mat3 arithmetic (ref_generate_case: Mat3::diagonal,
    matmul, inverse_adjugate from the unmodified mat3.cpp) and the C restatement,
    bit for bit, for every path x transform over the reference grid."""
    deltas = np.array(eig.default_delta_grid() + [0.0, 1e-14, 0.5, 3.0])
    R = U.ref()
    for gamma in (1e-3, 0.75):
        for path, pi in eig.PATHS.items():
            for kind, ki in eig.TRANSFORMS.items():
                got = eig.generate_case(path, kind, deltas, gamma=gamma).cpu().numpy()
                want = np.empty((deltas.size, 9))
                assert R.ref_generate_case(pi, ki, U.ctypes_double(gamma), U.ptr(deltas), U.S(deltas.size),
                                           U.ptr(want)) == 0
                assert U.bit_equal(got, want).all(), (path, kind, gamma)
                port = np.empty((deltas.size, 9))
                U.port().orc_generate_case(pi, ki, U.ctypes_double(gamma), U.ptr(deltas), U.S(deltas.size),
                                           U.ptr(port))
                assert U.bit_equal(port, want).all(), (path, kind, gamma)
    with pytest.raises(ValueError):
        eig.generate_case("D1", "U2", deltas, gamma=0.0)


def test_reference_eigensolver_known_answers():
    """proj/tests/test_eigensolver.cpp:54-69, 130-137 on the device:
    U1 similarity within 100 kappa2 ||A||_F eps; the D2/U1/1e-14 perf matrix
    within 1e-14 of the exact spectrum; eigvalss(diag(1,2,3)) within 12 eps."""
    from tests import _exact

    u1 = np.array([[1, -1, 1], [1, 1, 1], [-1, -1, 1]], dtype=np.float64)
    a = eig.generate_case("D1", "U1", [1.0]).cpu().numpy()  # U1 diag(1,1,2) U1^-1
    a2 = _mm(_mm(u1[None], np.diag([-1.0, 1.0, 2.0])[None]), _inv_adj(u1[None])[0]).reshape(1, 9)
    lam = eig.eigvals(a2).lam[0]
    kappa2 = np.linalg.cond(u1, 2)
    assert np.abs(lam - [-1, 1, 2]).max() <= 100 * kappa2 * np.sqrt((a2 * a2).sum()) * 2.0 ** -53
    pm = eig.generate_case("D2", "U1", [1e-14]).cpu().numpy()
    ex = [float(x) for x in _exact.exact_spectrum(pm[0])]
    assert np.abs(eig.eigvals(pm).lam[0] - ex).max() <= 1e-14
    lam_s = eig.eigvalss(np.diag([1.0, 2.0, 3.0])).lam[0]
    assert np.abs(lam_s - [1, 2, 3]).max() <= 12 * 2.0 ** -53
    assert a.shape == (1, 9)


def test_random_bit_patterns():
    """Uniformly random 64-bit patterns as entries (NaN payloads, subnormals,
    infinities, extreme exponents), alone and mixed row-wise with moderate
    entries so warps straddle all three tiers."""
    rng = np.random.default_rng(91)
    n = 1 << 18
    bits = rng.integers(0, 2 ** 63, size=(n, 9), dtype=np.int64) * rng.choice([1, -1], size=(n, 9))
    a = bits.view(np.float64).copy()
    mod = rng.standard_normal((n, 9))
    pick = rng.random((n, 9)) < 0.7
    a[n // 2:] = np.where(pick[n // 2:], mod[n // 2:], a[n // 2:])  # mostly-moderate rows
    lam, inv, flags = _run(a)
    _assert_parity(a, lam, inv, flags, "random-bits")


def test_native_cxx_driver_runs(tmp_path):
    """tools/native/eig33_bench.cpp: the C ABI driven from plain C++ (device
    and host-buffer entry points agree)."""
    exe = tmp_path / "eig33_bench"
    so_dir = os.path.join(U.ROOT, "paper_2511_00292_b200")
    r = subprocess.run(["g++", "-O2", "-std=c++17", "-I", os.path.join(U.ROOT, "include"),
                        os.path.join(U.ROOT, "tools", "native", "eig33_bench.cpp"),
                        os.path.join(so_dir, "_eig33cuda.so"), "-Wl,-rpath," + so_dir,
                        "-I/usr/local/cuda/include", "-L/usr/local/cuda/lib64", "-lcudart", "-o", str(exe)],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    out = subprocess.run([str(exe), "3", "18", "3"], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "agree on record 0: yes" in out.stdout
