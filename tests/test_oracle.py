"""Pins of the CPU oracle against things other than itself (no GPU needed).

Each test names the PAPER.md passage or the mathematical fact it relies on.
A plausible mistake in oracle/spa_oracle.c (dropped term, wrong index, swapped
operand, wrong table-size inequality, lowbnd off by one) fails one of these.
"""
import json
import os

import numpy as np
import pytest

import oracle
import synth


def _csr(d):
    return synth.CSR(d["nrows"], d["ncols"], np.array(d["row_ptr"], np.int64),
                     np.array(d["col"], np.int32), np.array(d["val"], np.float64))


def _dense_bruteforce(A, B):
    """Triple loop over the dense definition C_ij = sum_k A_ik B_kj (k ascending)."""
    Ad, Bd = A.to_dense(), B.to_dense()
    m, n = Ad.shape
    k = Bd.shape[1]
    C = [[0.0] * k for _ in range(m)]
    present = [[False] * k for _ in range(m)]
    for i in range(m):
        for kk in range(n):
            if Ad[i, kk] == 0.0:
                continue
            for j in range(k):
                if Bd[kk, j] == 0.0:
                    continue
                if present[i][j]:
                    C[i][j] = C[i][j] + Ad[i, kk] * Bd[kk, j]
                else:
                    C[i][j] = Ad[i, kk] * Bd[kk, j]
                    present[i][j] = True
    return np.array(C), np.array(present)


def _to_dense(m, k, rp, col, val):
    d = np.zeros((m, k))
    p = np.zeros((m, k), bool)
    for i in range(m):
        for t in range(rp[i], rp[i + 1]):
            assert not p[i, col[t]], "duplicate column in a row"
            d[i, col[t]] = val[t]
            p[i, col[t]] = True
    return d, p


# ---------------------------------------------------------------- golden files
def test_worked_example(golden_dir):
    g = json.load(open(os.path.join(golden_dir, "worked_2x2.json")))
    A, B = _csr(g["A"]), _csr(g["B"])
    rp, col, val = oracle.spgemm(A, B)
    assert rp.tolist() == g["C"]["row_ptr"]
    assert col.tolist() == g["C"]["col"]
    assert val.tolist() == g["C"]["val"]
    f, tot = oracle.flop(A, B)
    assert f.tolist() == g["flop"] and tot == sum(g["flop"])
    assert oracle.row_nnz(A, B).tolist() == g["row_nnz"]


def test_table_size_rule(golden_dir):
    g = json.load(open(os.path.join(golden_dir, "table_size.json")))
    for c in g["cases"]:
        assert oracle.table_size(c["flop"], c["ncols"]) == c["size"], c


def test_partition_examples(golden_dir):
    g = json.load(open(os.path.join(golden_dir, "partition.json")))
    for c in g["cases"]:
        assert oracle.rows_to_threads(np.array(c["flop"]), c["tnum"]).tolist() == c["offset"]


# ---------------------------------------------------------------- brute force
@pytest.mark.parametrize("seed", range(12))
def test_dense_bruteforce_bitexact(seed):
    """Sorted inputs: the SPA's canonical order equals the dense k-ascending
    sum, so values must agree bit for bit; structure = nonzero pattern for
    positive values."""
    rng = np.random.default_rng(seed)
    m, n, k = rng.integers(0, 14, size=3)
    A = synth.random_sparse(int(m), int(n), 0.3, seed, 0.5, 1.5, empty_rows=0.2)
    B = synth.random_sparse(int(n), int(k), 0.3, seed + 100, 0.5, 1.5, empty_rows=0.2)
    rp, col, val = oracle.spgemm(A, B)
    D, P = _to_dense(A.nrows, B.ncols, rp, col, val)
    Db, Pb = _dense_bruteforce(A, B)
    assert (P == Pb).all()
    assert (D == Db).all()
    for i in range(A.nrows):  # sorted output
        assert np.all(np.diff(col[rp[i]:rp[i + 1]]) > 0)


@pytest.mark.parametrize("seed", range(4))
def test_numpy_dense_midsize(seed):
    A = synth.random_sparse(90, 70, 0.08, seed, 0.0, 1.0)
    B = synth.random_sparse(70, 110, 0.08, seed + 1, 0.0, 1.0)
    rp, col, val = oracle.spgemm(A, B)
    D, P = _to_dense(90, 110, rp, col, val)
    ref = A.to_dense() @ B.to_dense()
    pat = (A.to_dense() != 0).astype(int) @ (B.to_dense() != 0).astype(int) > 0
    assert (P == pat).all()
    np.testing.assert_allclose(D, ref, rtol=1e-13, atol=0)


def test_unsorted_inputs_same_product():
    """Hash SpGEMM accepts 'Any' input order (Tab:summary)."""
    A = synth.random_sparse(60, 50, 0.1, 3, 0.5, 1.5)
    B = synth.random_sparse(50, 40, 0.1, 4, 0.5, 1.5)
    r1 = oracle.spgemm(A, B)
    r2 = oracle.spgemm(synth.shuffle_within_rows(A, 5), synth.shuffle_within_rows(B, 6))
    assert (r1[0] == r2[0]).all() and (r1[1] == r2[1]).all()
    np.testing.assert_allclose(r1[2], r2[2], rtol=1e-14)


def test_cancellation_kept():
    """Reading R1: structure is value-blind (symbolic inserts keys)."""
    A = synth.CSR(1, 2, np.array([0, 2], np.int64), np.array([0, 1], np.int32),
                  np.array([1.0, 1.0]))
    B = synth.CSR(2, 1, np.array([0, 1, 2], np.int64), np.array([0, 0], np.int32),
                  np.array([1.0, -1.0]))
    rp, col, val = oracle.spgemm(A, B)
    assert rp.tolist() == [0, 1] and col.tolist() == [0] and val.tolist() == [0.0]


def test_empty_shapes():
    E = synth.CSR(0, 5, np.zeros(1, np.int64), np.zeros(0, np.int32), np.zeros(0))
    B = synth.random_sparse(5, 3, 0.5, 1)
    rp, col, val = oracle.spgemm(E, B)
    assert rp.tolist() == [0] and len(col) == 0
    Z = synth.CSR(4, 5, np.zeros(5, np.int64), np.zeros(0, np.int32), np.zeros(0))
    rp, col, val = oracle.spgemm(Z, B)
    assert rp.tolist() == [0] * 5
    with pytest.raises(AssertionError):
        oracle.spgemm(B, B)  # 5x3 * 5x3: dimension mismatch


# ---------------------------------------------------------------- identities
def test_identity_bitexact():
    A = synth.er_poisson(300, 8.0, 11)
    I = synth.identity(300)
    for X, Y, ref in ((A, I, A), (I, A, A)):
        rp, col, val = oracle.spgemm(X, Y)
        assert (rp == ref.row_ptr).all() and (col == ref.col).all() and (val == ref.val).all()


def test_flop_by_outer_product_count():
    """flop = sum_k colcount_A(k) * rowcount_B(k) (a different formula than the
    row-wise loop of P:252-259); also nnz(C) <= flop and nnz(c_i) <= min(flop_i, ncols)."""
    A = synth.random_sparse(80, 60, 0.1, 21, empty_rows=0.1)
    B = synth.random_sparse(60, 70, 0.1, 22)
    f, tot = oracle.flop(A, B)
    colcnt = np.bincount(A.col, minlength=60)
    assert tot == int((colcnt * np.diff(B.row_ptr)).sum())
    nz = oracle.row_nnz(A, B)
    assert (nz <= np.minimum(f, B.ncols)).all()
    assert nz.sum() <= tot


def test_rowsum_identity():
    """C*1 = A*(B*1) within fp rounding for any values."""
    A, B, _ = synth.workload("c1_er4096", scale=9)
    rp, col, val = oracle.spgemm(A, B)
    lhs = np.bincount(np.repeat(np.arange(A.nrows), np.diff(rp)), weights=val, minlength=A.nrows)
    bsum = np.array([B.val[B.row_ptr[k]:B.row_ptr[k + 1]].sum() for k in range(B.nrows)])
    rhs = np.array([(A.val[A.row_ptr[i]:A.row_ptr[i + 1]] * bsum[A.col[A.row_ptr[i]:A.row_ptr[i + 1]]]).sum()
                    for i in range(A.nrows)])
    np.testing.assert_allclose(lhs, rhs, rtol=1e-12)


# ---------------------------------------------------------------- closed forms
def _c1(u, v, g, unit=True):
    d = abs(u - v)
    if d == 0:
        return 2 if (u == 0 or u == g - 1) else 3
    if d == 1:
        return 2
    if d == 2:
        return 1
    return 0


@pytest.mark.parametrize("g", [4, 5, 7])
def test_stencil_closed_forms(g):
    A = synth.stencil27(g, 1)
    assert A.nnz == (3 * g - 2) ** 3
    f, tot = oracle.flop(A, A)
    assert tot == (9 * g - 10) ** 3
    nz = oracle.row_nnz(A, A)
    assert nz.sum() == (5 * g - 6) ** 3
    # unit values: C(i,j) = prod_d c1(x_d, y_d)
    U = synth.CSR(A.nrows, A.ncols, A.row_ptr, A.col, np.ones(A.nnz))
    rp, col, val = oracle.spgemm(U, U)
    for i in range(0, A.nrows, 7):
        xi = (i % g, (i // g) % g, i // (g * g))
        for t in range(rp[i], rp[i + 1]):
            j = int(col[t])
            xj = (j % g, (j // g) % g, j // (g * g))
            assert val[t] == _c1(xi[0], xj[0], g) * _c1(xi[1], xj[1], g) * _c1(xi[2], xj[2], g)


@pytest.mark.parametrize("n", [3, 4, 7, 30])
def test_complete_graph_LU(n):
    G = synth.complete_graph(n)
    L, U = synth.tril_strict(G), synth.triu_strict(G)
    rp, col, val = oracle.spgemm(L, U)
    assert rp[-1] == (n - 1) ** 2
    D, P = _to_dense(n, n, rp, col, val)
    for i in range(n):
        for j in range(n):
            assert D[i, j] == min(i, j)
    f, tot = oracle.flop(L, U)
    assert tot == (n - 1) * n * (2 * n - 1) // 6
    assert oracle.triangle_count(L, U, G) == n * (n - 1) * (n - 2) // 6


def test_triangles_tree_and_k3():
    # a path (tree) has no triangle; K3 has one
    n = 10
    P = synth.from_coo(n, n, np.r_[np.arange(n - 1), np.arange(1, n)],
                       np.r_[np.arange(1, n), np.arange(n - 1)])
    assert oracle.triangle_count(synth.tril_strict(P), synth.triu_strict(P), P) == 0
    K3 = synth.complete_graph(3)
    assert oracle.triangle_count(synth.tril_strict(K3), synth.triu_strict(K3), K3) == 1


@pytest.mark.parametrize("seed", range(3))
def test_triangles_bruteforce(seed):
    rng = np.random.default_rng(seed)
    n = 40
    adj = rng.random((n, n)) < 0.2
    adj = np.triu(adj, 1)
    adj = adj | adj.T
    r, c = np.nonzero(adj)
    G = synth.from_coo(n, n, r, c)
    brute = sum(1 for a in range(n) for b in range(a + 1, n) for c_ in range(b + 1, n)
                if adj[a, b] and adj[b, c_] and adj[a, c_])
    L, U = synth.tril_strict(G), synth.triu_strict(G)
    assert oracle.triangle_count(L, U, G) == brute
    assert oracle.triangle_count(L, U, G, block_rows=7) == brute
    # L*U is symmetric (L = U^T) with diagonal = nnz(L row i)
    rp, col, val = oracle.spgemm(L, U)
    D, P = _to_dense(n, n, rp, col, val)
    assert (D == D.T).all() and (P == P.T).all()
    assert (np.diag(D) == np.diff(L.row_ptr)).all()


def _dense_pattern(M):
    D = np.zeros((M.nrows, M.ncols), dtype=bool)
    rows = np.repeat(np.arange(M.nrows), np.diff(M.row_ptr))
    D[rows, M.col[M.row_ptr[0]:M.row_ptr[-1]]] = True
    return D


@pytest.mark.parametrize("seed", range(3))
def test_degree_relabel_definition(seed):
    """P:604 reordering: G' = P G P^T (dense indexing), degrees nondecreasing
    along the new ids with ties by old id, L'/U' the strict triangles, sorted
    rows; the triangle count is invariant (brute force)."""
    rng = np.random.default_rng(100 + seed)
    n = 45
    adj = np.triu(rng.random((n, n)) < 0.15, 1)
    adj[0, 1:] |= rng.random(n - 1) < 0.6  # one hub
    adj = np.triu(adj, 1)
    adj = adj | adj.T
    r, c = np.nonzero(adj)
    G = synth.from_coo(n, n, r, c)
    perm, L2, U2, G2 = oracle.degree_relabel(G)
    assert sorted(perm.tolist()) == list(range(n))
    deg = adj.sum(1)
    key = [(deg[v], v) for v in perm]
    assert key == sorted(key)
    D2 = _dense_pattern(G2)
    assert (D2 == adj[np.ix_(perm, perm)]).all()
    assert (_dense_pattern(L2) == np.tril(D2, -1)).all()
    assert (_dense_pattern(U2) == np.triu(D2, 1)).all()
    for M in (L2, U2, G2):
        for i in range(n):
            row = M.col[M.row_ptr[i]:M.row_ptr[i + 1]]
            assert (np.diff(row) > 0).all()
    brute = sum(1 for a in range(n) for b in range(a + 1, n) for c_ in range(b + 1, n)
                if adj[a, b] and adj[b, c_] and adj[a, c_])
    assert oracle.triangle_count(L2, U2, G2) == brute
    # the hub goes last
    assert perm[-1] == int(np.argmax(deg)) or deg[perm[-1]] == deg.max()


@pytest.mark.parametrize("n", [5, 33])
def test_degree_relabel_star_closed_form(n):
    """Star K_{1,n-1} with the centre at id 0: natural-order L*U has (n-1)^2
    products (every leaf row meets the centre's U row); degree order puts the
    centre last and leaves n-1 products; no triangles either way."""
    r = np.r_[np.zeros(n - 1, int), np.arange(1, n)]
    c = np.r_[np.arange(1, n), np.zeros(n - 1, int)]
    G = synth.from_coo(n, n, r, c)
    L, U = synth.tril_strict(G), synth.triu_strict(G)
    assert oracle.flop(L, U)[1] == (n - 1) ** 2
    perm, L2, U2, G2 = oracle.degree_relabel(G)
    assert perm[-1] == 0 and list(perm[:-1]) == list(range(1, n))
    assert oracle.flop(L2, U2)[1] == n - 1
    assert oracle.triangle_count(L, U, G) == 0 == oracle.triangle_count(L2, U2, G2)


def test_degree_relabel_complete_graph_identity():
    """K_n: all degrees equal, so the order is the identity (ties by id)."""
    G = synth.complete_graph(9)
    perm, L2, U2, G2 = oracle.degree_relabel(G)
    assert list(perm) == list(range(9))
    L = synth.tril_strict(G)
    assert (L2.row_ptr == L.row_ptr).all() and (L2.col == L.col).all()


def test_tallskinny_columns():
    """C(:, j) = A(:, r_j) exactly when B has one 1.0 per column (config 4)."""
    A = synth.symmetrise_pattern(synth.rmat(8, 8, 5))
    B = synth.frontier(A.nrows, 64, 6)
    rp, col, val = oracle.spgemm(A, B)
    D, P = _to_dense(A.nrows, 64, rp, col, val)
    Ad = A.to_dense()
    rows_of_col = B.to_dense().argmax(axis=0)
    for j in range(64):
        assert (D[:, j] == Ad[:, rows_of_col[j]]).all()
    f, tot = oracle.flop(A, B)
    assert rp[-1] == tot  # CR = 1


def test_row_blocks_concatenate():
    A, B, _ = synth.workload("c3_rmat20", scale=9)
    rp, col, val = oracle.spgemm(A, B)
    parts = [oracle.spgemm(A, B, r0, min(A.nrows, r0 + 77)) for r0 in range(0, A.nrows, 77)]
    assert (np.concatenate([p[1] for p in parts]) == col).all()
    assert (np.concatenate([p[2] for p in parts]) == val).all()
    nz = np.concatenate([np.diff(p[0]) for p in parts])
    assert (nz == np.diff(rp)).all()


# ---------------------------------------------------------------- partition
@pytest.mark.parametrize("seed", range(6))
def test_partition_bound(seed):
    rng = np.random.default_rng(seed)
    m = int(rng.integers(1, 500))
    f = rng.integers(0, 1000, size=m) * (rng.random(m) < 0.7)
    for t in (1, 2, 3, 8, 600):
        off = oracle.rows_to_threads(f, t)
        ps = np.r_[0, np.cumsum(f)]
        assert off[0] == 0 and off[-1] == m and (np.diff(off) >= 0).all()
        tot = int(ps[-1])
        for tid in range(1, t):  # lowbnd semantics vs numpy searchsorted
            assert off[tid] == np.searchsorted(ps, (tot * tid) // t, side="left")
        work = ps[off[1:]] - ps[off[:-1]]
        assert work.max(initial=0) <= -(-tot // t) + f.max(initial=0)
