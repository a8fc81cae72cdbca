"""The reference-module drop-in (paper_2511_00292_b200.eig33): names, input
parsing and the EigenTriple type, checked without a GPU.  The numbers are
checked on the GPU in test_compat_gpu.py."""
import numpy as np
import pytest

from paper_2511_00292_b200 import eig33

# bindings/module.cpp:98-104
REFERENCE_ALL = ["EigenTriple", "eps_mach", "eigvals", "eigvalss", "eigvals_naive", "i1", "j2_stable",
                 "j2_naive", "j2_tensor", "j3_stable", "j3_naive", "j3_tensor", "disc_stable",
                 "disc_naive", "jacobian_j2", "jacobian_j3", "jacobian_disc"]


def test_public_surface_matches_reference_module():
    assert eig33.__all__ == REFERENCE_ALL
    for name in REFERENCE_ALL:
        assert hasattr(eig33, name), name
    assert eig33.eps_mach == 2.0 ** -53  # tests/python/test_smoke.py:88-89


def test_to_mat_accepts_flat_and_nested():
    flat, s1 = eig33._parse([0.5, 0.25, -1, 0.125, -3, 2, 0, 1, 4])
    nested, s2 = eig33._parse([[0.5, 0.25, -1], [0.125, -3, 2], [0, 1, 4]])
    assert s1 and s2 and (flat == nested).all() and flat.shape == (1, 9)
    tup, _ = eig33._parse(((1, 2, 3), (4, 5, 6), (7, 8, 9)))
    assert tup.tolist() == [[1, 2, 3, 4, 5, 6, 7, 8, 9]]


@pytest.mark.parametrize("bad", [[1, 2, 3], "abcdefghi", 5, None, [[1, 2], [3, 4], [5, 6]],
                                 [1, 2, 3, 4], [[1, 2, 3], [4, 5, 6], 7], [1, 2, 3, 4, 5, 6, 7, 8, "x"]])
def test_to_mat_rejects_like_the_binding(bad):
    """module.cpp:16-39 throws std::invalid_argument -> ValueError
    (tests/python/test_smoke.py:92-97 for the 3-entry case)."""
    with pytest.raises(ValueError):
        eig33._parse(bad)


def test_arrays_single_and_batch():
    _, single = eig33._parse(np.eye(3))
    assert single
    _, single = eig33._parse(np.zeros(9))
    assert single
    recs, single = eig33._parse(np.zeros((5, 3, 3)))
    assert not single and recs.shape == (5, 9)
    recs, single = eig33._parse(np.zeros((1, 9)))
    assert not single and recs.shape == (1, 9)


def test_eigen_triple_behaves_like_the_bound_struct():
    t = eig33.EigenTriple(1.0, 2.0, 3.0)
    assert len(t) == 3 and list(t) == [1.0, 2.0, 3.0] and t[-1] == 3.0 and t[-3] == 1.0
    with pytest.raises(IndexError):
        t[3]
    assert (t.lambda1, t.lambda2, t.lambda3, t.non_real_advisory) == (1.0, 2.0, 3.0, False)
    assert repr(t) == "EigenTriple(1.0, 2.0, 3.0)"
    assert repr(eig33.EigenTriple(-1.5, 0.0, 2.0, True)) == "EigenTriple(-1.5, 0.0, 2.0, non_real_advisory=True)"
