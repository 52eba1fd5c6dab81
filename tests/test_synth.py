"""Generators (shared by oracle and CUDA path): determinism and shape facts."""
import numpy as np

import synth


def test_determinism():
    a = synth.rmat(10, 16, 3)
    b = synth.rmat(10, 16, 3)
    assert (a.row_ptr == b.row_ptr).all() and (a.col == b.col).all() and (a.val == b.val).all()
    a.check()


def test_rmat_quadrants():
    """Top-level quadrant frequencies of the draws follow a,b,c,d."""
    r, c = synth.rmat_edges(12, 16, 0.57, 0.19, 0.19, 9)
    half = 1 << 11
    q = (r >= half).astype(int) * 2 + (c >= half).astype(int)
    freq = np.bincount(q, minlength=4) / len(q)
    np.testing.assert_allclose(freq, [0.57, 0.19, 0.19, 0.05], atol=0.005)


def test_stencil_counts():
    A = synth.stencil27(6, 1)
    A.check()
    assert A.nnz == 16 ** 3
    assert (A.val >= 0.5).all() and (A.val < 1.5).all()


def test_symmetrise_and_triangles():
    R = synth.rmat(9, 8, 2)
    G = synth.symmetrise_pattern(R, drop_diagonal=True)
    D = G.to_dense()
    assert (D == D.T).all() and (np.diag(D) == 0).all()
    L, U = synth.tril_strict(G), synth.triu_strict(G)
    assert L.nnz + U.nnz == G.nnz
    assert (L.to_dense() == U.to_dense().T).all()


def test_frontier():
    B = synth.frontier(1000, 64, 4)
    B.check()
    assert B.nnz == 64 and (np.sort(B.col) == np.arange(64)).all()


def test_er_rows():
    A = synth.er_poisson(512, 8.0, 1)
    A.check()
    assert abs(A.nnz / 512 - 8.0) < 0.6
    for i in range(512):
        c, _ = A.row(i)
        assert (np.diff(c) > 0).all()


def test_shuffle_keeps_rows():
    A = synth.random_sparse(30, 30, 0.3, 1)
    S = synth.shuffle_within_rows(A, 2)
    for i in range(30):
        assert sorted(S.row(i)[0].tolist()) == A.row(i)[0].tolist()
