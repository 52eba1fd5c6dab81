"""GPU parity: the CUDA path (through the C ABI) vs the oracle on the same
seeded inputs.  Every test here needs a B200 (marker `gpu`)."""
import numpy as np
import pytest

import oracle
import synth
from parity import compare, compare_rows, gpu_vs_oracle, sampled_rows

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def spg():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1804_01698_b200 as m
    from paper_1804_01698_b200 import build
    build.build()
    return m


@pytest.fixture(scope="module")
def ctx(spg):
    return spg.Context()


# ------------------------------------------------------------------ small
@pytest.mark.parametrize("sorted_out", [True, False])
def test_worked_example(spg, ctx, sorted_out):
    A = synth.CSR(2, 2, np.array([0, 1, 3], np.int64), np.array([0, 0, 1], np.int32),
                  np.array([1.0, 2.0, 3.0]))
    B = synth.CSR(2, 2, np.array([0, 1, 2], np.int64), np.array([1, 0], np.int32),
                  np.array([4.0, 5.0]))
    gpu_vs_oracle(A, B, sorted_out, ctx=ctx, what="2x2")


@pytest.mark.parametrize("seed", range(10))
@pytest.mark.parametrize("sorted_out", [True, False])
def test_random_shapes(spg, ctx, seed, sorted_out):
    rng = np.random.default_rng(seed)
    m, n, k = (int(x) for x in rng.integers(1, 300, size=3))
    A = synth.random_sparse(m, n, float(rng.uniform(0.001, 0.1)), seed, 0.0, 1.0, empty_rows=0.2)
    B = synth.random_sparse(n, k, float(rng.uniform(0.001, 0.1)), seed + 50, 0.0, 1.0,
                            empty_rows=0.1)
    gpu_vs_oracle(A, B, sorted_out, ctx=ctx, what=f"random{seed}")


def test_empty_and_degenerate(spg, ctx):
    for (m, n, k) in [(0, 5, 7), (5, 0, 7), (5, 7, 0), (1, 1, 1)]:
        A = synth.random_sparse(m, n, 0.5, 1)
        B = synth.random_sparse(n, k, 0.5, 2)
        gpu_vs_oracle(A, B, True, ctx=ctx, what=f"{m}x{n}x{k}")
    Z = synth.CSR(6, 4, np.zeros(7, np.int64), np.zeros(0, np.int32), np.zeros(0))
    gpu_vs_oracle(Z, synth.random_sparse(4, 9, 0.5, 3), True, ctx=ctx, what="nnz(A)=0")


def test_dimension_mismatch(spg, ctx):
    A = spg.DeviceCSR.from_host(synth.random_sparse(4, 5, 0.5, 1))
    with pytest.raises(ValueError):
        spg.spgemm(A, A, ctx=ctx)
    from paper_1804_01698_b200 import _lib
    rp = torch.zeros(5, dtype=torch.int64, device="cuda")
    with pytest.raises(_lib.SpgError, match="DIM_MISMATCH"):
        _lib.spg_symbolic(ctx.handle, A.c(), A.c(), rp.data_ptr(), 0)


def test_numeric_without_symbolic_is_state_error(spg):
    from paper_1804_01698_b200 import _lib
    c2 = spg.Context()
    A = spg.DeviceCSR.from_host(synth.random_sparse(4, 4, 0.5, 1))
    rp = torch.zeros(5, dtype=torch.int64, device="cuda")
    with pytest.raises(_lib.SpgError, match="STATE"):
        _lib.spg_numeric(c2.handle, A.c(), A.c(), rp.data_ptr(), 0, 0, True, 0)


def test_numeric_with_other_arrays_is_state_error(spg):
    """The plan is keyed on every array the symbolic phase read: a numeric call
    whose A or B carries another col_idx array is refused."""
    from paper_1804_01698_b200 import _lib
    c2 = spg.Context()
    A = spg.DeviceCSR.from_host(synth.random_sparse(40, 40, 0.2, 3))
    rp, nnz, _ = spg.spg_symbolic(A, A, c2)
    A2 = spg.DeviceCSR(A.nrows, A.ncols, A.row_ptr, A.col.clone(), A.val)
    for a, b in ((A2, A), (A, A2)):
        with pytest.raises(_lib.SpgError, match="STATE"):
            spg.spg_numeric(a, b, rp, nnz, ctx=c2)
    C = spg.spg_numeric(A, A, rp, nnz, ctx=c2)  # the matching call still runs
    compare(*C.to_host(), *oracle.spgemm(synth.random_sparse(40, 40, 0.2, 3),
                                         synth.random_sparse(40, 40, 0.2, 3)), True, "plan keyed")


def test_identity_bitexact(spg, ctx):
    A = synth.er_poisson(2000, 8.0, 5)
    I = synth.identity(2000)
    for X, Y in ((A, I), (I, A)):
        C = spg.spgemm(spg.DeviceCSR.from_host(X), spg.DeviceCSR.from_host(Y), True, ctx)
        rp, col, val = C.to_host()
        assert (rp == A.row_ptr).all() and (col == A.col).all() and (val == A.val).all()


def test_unsorted_input_order(spg, ctx):
    A, B, _ = synth.workload("c3_rmat20", scale=11)
    As, Bs = synth.shuffle_within_rows(A, 1), synth.shuffle_within_rows(B, 2)
    for so in (True, False):
        gpu_vs_oracle(As, Bs, so, ctx=ctx, what="shuffled input")


# ------------------------------------------------------------------ bins
def _boundary_specs():
    specs = [(0, 0)]
    for T in [128, 1024, 2048, 4096, 8192, 16384, 32768, 65536]:
        for f in (T - 1, T, T + 1):
            specs.append((f, 37))          # symbolic-bin boundaries, low nnz
    for h in [16, 128, 512, 1024, 2048, 4096, 8192, 16384]:
        for n in (h - 1, h, h + 1):
            specs.append((n, n))           # numeric-bin boundaries, CR = 1
            specs.append((3 * n + 1, n))   # same nnz, CR ~ 3
    specs += [(200000, 60000), (50000, 50000), (1, 1), (2, 1), (33, 33)]
    return specs


@pytest.mark.parametrize("sorted_out", [True, False])
@pytest.mark.parametrize("shuffle", [False, True])
def test_bin_boundaries(spg, ctx, sorted_out, shuffle):
    A, B = synth.crafted_rows(_boundary_specs(), 1 << 17, 11, shuffle=shuffle)
    gpu_vs_oracle(A, B, sorted_out, ctx=ctx, what="bin boundaries")


@pytest.mark.parametrize("sorted_out", [True, False])
def test_wide_columns_global_tables(spg, ctx, sorted_out):
    """ncols > the smem bitmap limit: global-hash symbolic, multi-chunk rank sort."""
    specs = [(70000, 30000), (40000, 20000), (100, 100), (3000, 1000)]
    A, B = synth.crafted_rows(specs, 3_000_000, 12)
    gpu_vs_oracle(A, B, sorted_out, ctx=ctx, what="wide ncols")


@pytest.mark.parametrize("sorted_out", [True, False])
@pytest.mark.parametrize("shuffle", [False, True])
def test_column_parts(spg, ctx, sorted_out, shuffle):
    """Long rows over a 1M-column space: column-range parts with rank and width
    cuts (sorted B), or the global-hash fallback (shuffled B)."""
    specs = [(150000, 50000), (30000, 9000), (9000, 8193), (8193, 8193), (70000, 4097),
             (20000, 12000), (5, 5), (0, 0), (600000, 200000)]
    A, B = synth.crafted_rows(specs, 1_000_000, 14, shuffle=shuffle)
    gpu_vs_oracle(A, B, sorted_out, ctx=ctx, what="column parts")


def _tile_rows(tile_keys, ntiles, seed, overlap=3):
    """(A, B) with ONE row of A*B whose keys per 8192-column tile are exactly
    tile_keys (column-part cutter cases); B rows sorted, each key reached from
    1..overlap B rows (CR > 1)."""
    rng = np.random.default_rng(seed)
    cols = []
    for t, kcount in enumerate(tile_keys):
        if kcount:
            cols.append(t * 8192 + np.sort(rng.choice(8192, size=kcount, replace=False)))
    S = np.concatenate(cols).astype(np.int64)
    b_rows, b_cols = [], []
    for r in range(overlap):  # B row r holds every key with (key index % overlap) <= r
        keep = (np.arange(len(S)) % overlap) <= r
        b_rows.append(np.full(int(keep.sum()), r, np.int64))
        b_cols.append(S[keep])
    B = synth.from_coo(overlap, ntiles * 8192, np.concatenate(b_rows), np.concatenate(b_cols))
    B = synth.with_values(B, seed + 1, 0.5, 1.5)
    A = synth.from_coo(1, overlap, np.zeros(overlap, np.int64), np.arange(overlap))
    A = synth.with_values(A, seed + 2, 0.5, 1.5)
    return A, B


@pytest.mark.parametrize("tile_keys", [
    [0, 8192, 100],              # empty tile, then a full tile (> 4096 keys)
    [3000, 0, 5000, 500],        # empty tile between two (the advisor's case)
    [0, 0, 0, 6000, 0, 3000],    # leading empty tiles, heavy tile, trailing gap
    [2000, 100, 0, 4500, 2100, 2048, 1, 0, 0, 2047],
    [1500] * 6,                  # runs of tiles that fill a 2048-key part
])
@pytest.mark.parametrize("sorted_out", [True, False])
def test_part_cutter_tile_patterns(spg, ctx, tile_keys, sorted_out):
    """Column-tile part cuts (advisor r01 finding): a heavy tile always stands
    alone, runs of >= 2 tiles hold <= 2048 keys, parts start at nonempty
    tiles -- whatever the pattern of empty tiles.  Exact vs the oracle."""
    assert sum(tile_keys) > 8192  # a long row: column-tile parts
    A, B = _tile_rows(tile_keys, max(len(tile_keys), 8), 31)
    gpu_vs_oracle(A, B, sorted_out, ctx=ctx, what=f"tiles {tile_keys}")


@pytest.mark.parametrize("sorted_out", [True, False])
def test_signed_values_cancellation(spg, ctx, sorted_out):
    """Reading R1: numerically cancelled entries stay in the structure.  Rows
    of A pick pairs of B rows with equal patterns and equal values, with a_ik
    = +x and -x, so those entries of C sum to exactly 0.0 (two terms, any
    order) and must still be present.  Other entries mix signs: values within
    1e-12 of the sum of |terms| (the error bound of a signed sum), computed by
    the oracle on |A|*|B|."""
    rng = np.random.default_rng(5)
    n, k, m = 4000, 3000, 600
    B0 = synth.random_sparse(k // 2, n, 0.01, 8, -1.0, 1.0)
    # B = [B0; B0] (rows k/2 + r duplicate rows r)
    B = synth.CSR(k, n, np.r_[B0.row_ptr, B0.row_ptr[1:] + B0.row_ptr[-1]].astype(np.int64),
                  np.r_[B0.col, B0.col].astype(np.int32), np.r_[B0.val, B0.val])
    rows, cols, vals = [], [], []
    for i in range(m):
        picks = rng.choice(k // 2, size=int(rng.integers(1, 40)), replace=False)
        x = rng.uniform(0.5, 2.0, size=len(picks))
        ncancel = len(picks) // 2
        rows += [i] * (len(picks) + ncancel)
        cols += list(picks) + list(picks[:ncancel] + k // 2)
        vals += list(x) + list(-x[:ncancel])
    A = synth.from_coo(m, k, np.array(rows), np.array(cols), np.array(vals))
    import paper_1804_01698_b200 as spgm
    dA, dB = spgm.DeviceCSR.from_host(A), spgm.DeviceCSR.from_host(B)
    C = spgm.spgemm(dA, dB, sorted=sorted_out, ctx=ctx)
    g_rp, g_col, g_val = C.to_host()
    o_rp, o_col, o_val = oracle.spgemm(A, B)
    assert np.array_equal(g_rp - g_rp[0], o_rp)
    if not sorted_out:
        from parity import sort_rows
        g_col, g_val = sort_rows(g_rp, g_col, g_val)
    assert np.array_equal(g_col, o_col)
    absA = synth.CSR(A.nrows, A.ncols, A.row_ptr, A.col, np.abs(A.val))
    absB = synth.CSR(B.nrows, B.ncols, B.row_ptr, B.col, np.abs(B.val))
    _, a_col, mag = oracle.spgemm(absA, absB)
    assert np.array_equal(a_col, o_col)
    assert (np.abs(g_val - o_val) <= 1e-12 * mag).all()
    assert (o_val == 0.0).sum() > 100  # cancelled entries exist and are kept


@pytest.mark.parametrize("ncols", [1, 2, 16])
def test_small_ncols_cap(spg, ctx, ncols):
    """min(N_col, flop) cap of the table size: large flop, tiny ncols."""
    specs = [(5000, ncols), (40000, ncols), (7, min(7, ncols)), (100000, ncols)]
    A, B = synth.crafted_rows(specs, ncols, 13)
    gpu_vs_oracle(A, B, True, ctx=ctx, what=f"ncols={ncols}")


def test_dense_output_rows(spg, ctx):
    A = synth.random_sparse(40, 60, 0.9, 3, 0.5, 1.5)
    B = synth.random_sparse(60, 700, 0.5, 4, 0.5, 1.5)
    for so in (True, False):
        gpu_vs_oracle(A, B, so, ctx=ctx, what="dense rows")


# ------------------------------------------------------------------ plan
def test_plan_flop_and_table_size(spg, ctx):
    A, B = synth.crafted_rows(_boundary_specs(), 1 << 17, 21)
    dA, dB = spg.DeviceCSR.from_host(A), spg.DeviceCSR.from_host(B)
    rp, nnz, flop_tot = spg.spg_symbolic(dA, dB, ctx)
    f, t = spg.plan_export(ctx, A.nrows)
    of, otot = oracle.flop(A, B)
    assert flop_tot == otot
    assert (f.cpu().numpy() == of).all()
    ot = np.array([oracle.table_size(x, B.ncols) for x in of])
    assert (t.cpu().numpy() == ot).all()
    assert (np.diff(rp.cpu().numpy()) == oracle.row_nnz(A, B)).all()
    info = ctx.info()
    assert info["nnz_total"] == nnz and info["flop_total"] == otot


@pytest.mark.parametrize("nparts", [1, 2, 3, 8, 64])
def test_rows_to_parts(spg, ctx, nparts):
    A, B, _ = synth.workload("c3_rmat20", scale=12)
    offs, tot = spg.rows_to_parts(spg.DeviceCSR.from_host(A), spg.DeviceCSR.from_host(B),
                                  nparts, ctx)
    of, otot = oracle.flop(A, B)
    assert tot == otot
    assert offs == oracle.rows_to_threads(of, nparts).tolist()


# ------------------------------------------------------------------ configs
@pytest.mark.parametrize("sorted_out", [True, False])
def test_c1_er_full(spg, ctx, sorted_out):
    A, B, _ = synth.workload("c1_er4096")
    gpu_vs_oracle(A, B, sorted_out, ctx=ctx, what="C1")


@pytest.mark.parametrize("g", [8, 33])
@pytest.mark.parametrize("sorted_out", [True, False])
def test_c2_stencil_small(spg, ctx, g, sorted_out):
    A, B, _ = synth.workload("c2_stencil64", scale=g)
    gpu_vs_oracle(A, B, sorted_out, ctx=ctx, what=f"C2 g={g}")


@pytest.mark.parametrize("scale", [10, 14])
@pytest.mark.parametrize("sorted_out", [True, False])
def test_c3_rmat_small(spg, ctx, scale, sorted_out):
    A, B, _ = synth.workload("c3_rmat20", scale=scale)
    gpu_vs_oracle(A, B, sorted_out, ctx=ctx, what=f"C3 s{scale}")


def test_c4_tallskinny_small(spg, ctx):
    A, B, _ = synth.workload("c4_tallskinny", scale=14)
    gpu_vs_oracle(A, B, False, ctx=ctx, what="C4 s14")


@pytest.mark.parametrize("sorted_out", [False, True])
def test_c4_tallskinny_pruned(spg, ctx, sorted_out):
    """Scale 16 (nnz(A) > 2^20, B 99.9% empty rows): the plan runs on the
    pruned A' -- structure and values still exact vs the oracle, and a second
    numeric on the same plan with other A values uses the new values."""
    A, B, _ = synth.workload("c4_tallskinny", scale=16)
    assert A.nnz >= (1 << 20)
    gpu_vs_oracle(A, B, sorted_out, ctx=ctx, what="C4 s16 pruned")
    A2 = synth.with_values(A, 77, 0.5, 1.5)
    dA, dB = spg.DeviceCSR.from_host(A), spg.DeviceCSR.from_host(B)
    dA2 = spg.DeviceCSR(A.nrows, A.ncols, dA.row_ptr, dA.col,
                        torch.from_numpy(A2.val).to(dA.row_ptr.device))
    rp, nnz, _ = spg.spg_symbolic(dA, dB, ctx)           # plan on A (values unused)
    C = spg.spg_numeric(dA2, dB, rp, nnz, sorted_out, ctx)  # same structure, new values
    from parity import compare
    compare(*C.to_host(), *oracle.spgemm(A2, B), sorted_out, "C4 s16 pruned, new values")


@pytest.mark.parametrize("scale", [10, 14])
def test_c5_triangles_small(spg, ctx, scale):
    L, U, ex = synth.workload("c5_triangle", scale=scale)
    G = ex["G"]
    gpu_vs_oracle(L, U, True, ctx=ctx, what=f"C5 s{scale} L*U")
    want = oracle.triangle_count(L, U, G)
    dL, dU, dG = (spg.DeviceCSR.from_host(x) for x in (L, U, G))
    for so in (False, True):
        assert spg.triangle_count(dL, dU, dG, sorted=so, ctx=ctx) == want
    # force several row blocks (streaming path)
    assert spg.triangle_count(dL, dU, dG, block_entries=max(1, L.nnz // 3), ctx=ctx) == want


def test_triangles_complete_graph(spg, ctx):
    n = 60
    G = synth.complete_graph(n)
    L, U = synth.tril_strict(G), synth.triu_strict(G)
    dL, dU, dG = (spg.DeviceCSR.from_host(x) for x in (L, U, G))
    assert spg.triangle_count(dL, dU, dG, ctx=ctx) == n * (n - 1) * (n - 2) // 6


# ------------------------------------------------------------------ fused mask
@pytest.mark.parametrize("scale", [10, 14])
def test_c5_triangles_fused(spg, ctx, scale):
    """Fused mask-and-sum (C never formed) vs the oracle's triangle count;
    scale 14 has G rows above the warp tier (bitmap tier)."""
    L, U, ex = synth.workload("c5_triangle", scale=scale)
    G = ex["G"]
    want = oracle.triangle_count(L, U, G)
    dL, dU, dG = (spg.DeviceCSR.from_host(x) for x in (L, U, G))
    assert spg.triangle_count_fused(dL, dU, dG, ctx=ctx) == want
    if scale == 14:
        assert int(np.diff(G.row_ptr).max()) > 256  # both tiers ran


def _relabel_vs_oracle(spg, ctx, G):
    perm, L2, U2, G2 = spg.degree_relabel(spg.DeviceCSR.from_host(G), ctx=ctx)
    o_perm, oL, oU, oG = oracle.degree_relabel(G)
    assert np.array_equal(perm.cpu().numpy(), o_perm)  # unique order: (degree, id)
    for d, o in ((L2, oL), (U2, oU), (G2, oG)):
        assert np.array_equal(d.row_ptr.cpu().numpy(), o.row_ptr)
        assert np.array_equal(d.col.cpu().numpy(), o.col)  # sorted rows, bit-exact
        assert (d.val.cpu().numpy() == 1.0).all()
    return L2, U2, G2


@pytest.mark.parametrize("scale", [10, 14])
def test_degree_relabel_parity(spg, ctx, scale):
    """P:604 reordering on the GPU vs the oracle (perm, L', U', G' exact), and
    the triangle count of the reordered split equals the natural-order count
    (oracle), fused and with C formed."""
    L, U, ex = synth.workload("c5_triangle", scale=scale)
    G = ex["G"]
    want = oracle.triangle_count(L, U, G)
    L2, U2, G2 = _relabel_vs_oracle(spg, ctx, G)
    assert spg.triangle_count_fused(L2, U2, G2, ctx=ctx) == want
    assert spg.triangle_count(L2, U2, G2, sorted=True, ctx=ctx) == want
    # the point of the reordering: far fewer products than the natural order
    _, f_nat = oracle.flop(L, U)
    _, f_deg = spg.rows_to_parts(L2, U2, 1, ctx)
    assert f_deg < f_nat


def test_degree_relabel_edge_cases(spg, ctx):
    # star (hub moves last), K_n (identity), a graph with isolated vertices,
    # an edgeless graph, a single vertex
    n = 40
    r = np.r_[np.zeros(n - 1, int), np.arange(1, n)]
    c = np.r_[np.arange(1, n), np.zeros(n - 1, int)]
    _relabel_vs_oracle(spg, ctx, synth.from_coo(n, n, r, c))
    _relabel_vs_oracle(spg, ctx, synth.complete_graph(50))
    iso = synth.from_coo(10, 10, np.array([2, 7, 7, 9]), np.array([7, 2, 9, 7]))
    _relabel_vs_oracle(spg, ctx, iso)
    _relabel_vs_oracle(spg, ctx, synth.from_coo(6, 6, np.array([], int), np.array([], int)))
    _relabel_vs_oracle(spg, ctx, synth.from_coo(1, 1, np.array([], int), np.array([], int)))
    _relabel_vs_oracle(spg, ctx, synth.from_coo(0, 0, np.array([], int), np.array([], int)))
    # errors: a diagonal entry; a non-symmetric pattern
    with pytest.raises(Exception):
        spg.degree_relabel(spg.DeviceCSR.from_host(
            synth.from_coo(3, 3, np.array([0, 1, 2, 1]), np.array([1, 0, 2, 2]))), ctx=ctx)
    with pytest.raises(Exception):
        spg.degree_relabel(spg.DeviceCSR.from_host(
            synth.from_coo(3, 3, np.array([0, 0]), np.array([1, 2]))), ctx=ctx)


def test_triangles_fused_complete_graph(spg, ctx):
    for n in (3, 60, 700):  # 700: G rows of 699 > the warp tier
        G = synth.complete_graph(n)
        L, U = synth.tril_strict(G), synth.triu_strict(G)
        dL, dU, dG = (spg.DeviceCSR.from_host(x) for x in (L, U, G))
        assert spg.triangle_count_fused(dL, dU, dG, ctx=ctx) == n * (n - 1) * (n - 2) // 6


@pytest.mark.parametrize("ncols", [5000, 2_000_000])
def test_masked_sum_random_values(spg, ctx, ncols):
    """General values: sum over pattern(G) of (A*B) vs the oracle's C and
    mask_sum; ncols 2M > the bitmap limit (binary-search tier)."""
    rng = np.random.default_rng(ncols)
    m, k = 300, 400
    A = synth.random_sparse(m, k, 0.05, 11, 0.0, 1.0)
    B = synth.random_sparse(k, ncols, min(0.5, 3000.0 / ncols), 12, 0.0, 1.0)
    o_rp, o_col, o_val = oracle.spgemm(A, B)
    # G: half of C's pattern per row plus random extra columns; some rows long
    rows, cols = [], []
    for i in range(m):
        ci = o_col[o_rp[i]:o_rp[i + 1]]
        keep = ci[rng.random(len(ci)) < 0.5]
        extra = rng.integers(0, ncols, size=int(rng.integers(0, 600 if i % 7 == 0 else 40)))
        cc = np.unique(np.r_[keep, extra]).astype(np.int64)
        rows.append(np.full(len(cc), i)); cols.append(cc)
    G = synth.from_coo(m, ncols, np.concatenate(rows), np.concatenate(cols))
    want = 0.0
    for i in range(m):  # oracle-side mask sum in fp64 (canonical order)
        ci, vi = o_col[o_rp[i]:o_rp[i + 1]], o_val[o_rp[i]:o_rp[i + 1]]
        g = G.col[G.row_ptr[i]:G.row_ptr[i + 1]]
        want += float(vi[np.isin(ci, g)].sum())
    dA, dB, dG = (spg.DeviceCSR.from_host(x) for x in (A, B, G))
    got = spg.masked_sum(dA, dB, dG, 0, ctx)
    assert abs(got - want) <= 1e-12 * abs(want), (got, want)


def test_validate(spg, ctx):
    from paper_1804_01698_b200 import _lib
    A = synth.random_sparse(50, 40, 0.2, 1)
    spg.validate(spg.DeviceCSR.from_host(A), True, ctx)
    bad = synth.CSR(A.nrows, A.ncols, A.row_ptr, A.col.copy(), A.val)
    bad.col[3] = 45
    with pytest.raises(_lib.SpgError, match="INDEX_RANGE"):
        spg.validate(spg.DeviceCSR.from_host(bad), False, ctx)
    S = synth.shuffle_within_rows(synth.random_sparse(50, 40, 0.5, 2), 3)
    spg.validate(spg.DeviceCSR.from_host(S), False, ctx)
    with pytest.raises(_lib.SpgError):
        spg.validate(spg.DeviceCSR.from_host(S), True, ctx)


def test_sorted_equals_sorted_unsorted(spg, ctx):
    A, B, _ = synth.workload("c3_rmat20", scale=13)
    dA = spg.DeviceCSR.from_host(A)
    Cs = spg.spgemm(dA, dA, True, ctx)
    Cu = spg.spgemm(dA, dA, False, ctx)
    rs, cs, vs = Cs.to_host()
    ru, cu, vu = Cu.to_host()
    compare(ru, cu, vu, rs, cs, vs, False, "sorted vs unsorted")


def test_row_range_view(spg, ctx):
    A, B, _ = synth.workload("c3_rmat20", scale=12)
    dA = spg.DeviceCSR.from_host(A)
    r0, r1 = 777, 2900
    C = spg.spgemm(dA.rows(r0, r1), dA, True, ctx)
    g = C.to_host()
    o = oracle.spgemm(A, B, r0, r1)
    compare(*g, *o, True, "row view")


# ------------------------------------------------------------------ full size
@pytest.mark.parametrize("sorted_out", [True, False])
def test_c2_full_size(spg, ctx, sorted_out):
    """BASELINE config 2 at full size, whole product vs the oracle."""
    A, B, _ = synth.workload("c2_stencil64")
    gpu_vs_oracle(A, B, sorted_out, ctx=ctx, what="C2 full")


@pytest.mark.slow
def test_c3_full_size_sampled(spg, ctx):
    """BASELINE config 3 at full size (C = 116 GB): sampled rows (heaviest +
    random) vs the oracle, and the row-sum identity over all rows."""
    A, B, _ = synth.workload("c3_rmat20")
    dA = spg.DeviceCSR.from_host(A)
    free, _ = torch.cuda.mem_get_info()
    of, otot = oracle.flop(A, B)
    for so in (False, True):
        C = spg.spgemm(dA, dA, so, ctx)
        assert ctx.info()["flop_total"] == otot
        rows = sampled_rows(A, B, of, nsample=150, seed=3, top=8)
        compare_rows(C, A, B, rows, so, what=f"C3 full sorted={so}")
        # row sums: C*1 vs A*(B*1) computed on the host from A, B (fp64)
        rp = C.row_ptr
        rs = torch.zeros(A.nrows, dtype=torch.float64, device="cuda")
        rp_h = rp.cpu().numpy()
        r0 = 0
        while r0 < A.nrows:  # row blocks of <= 2^28 entries (C3's C has 9.7e9)
            r1 = int(np.searchsorted(rp_h, rp_h[r0] + (1 << 28), side="right")) - 1
            r1 = min(max(r1, r0 + 1), A.nrows)
            lens = rp[r0 + 1:r1 + 1] - rp[r0:r1]
            idx = torch.repeat_interleave(torch.arange(r0, r1, device="cuda"), lens)
            rs.index_add_(0, idx, C.val[int(rp_h[r0]):int(rp_h[r1])])
            del idx
            r0 = r1
        bsum = np.bincount(np.repeat(np.arange(B.nrows), np.diff(B.row_ptr)), weights=B.val,
                           minlength=B.nrows)
        ref = np.bincount(np.repeat(np.arange(A.nrows), np.diff(A.row_ptr)),
                          weights=A.val * bsum[A.col], minlength=A.nrows)
        np.testing.assert_allclose(rs.cpu().numpy(), ref, rtol=1e-11, atol=1e-300)
        del C, rs
        torch.cuda.empty_cache()


@pytest.mark.parametrize("which", ["c2", "c3"])
def test_probe_stats(spg, ctx, which):
    """Collision-factor measurement (Eq:hash_est P:362):
    every mode inserts exactly the distinct keys of the measured rows (oracle
    row nnz), each insert costs >= 1 probe, and on the stencil the high-bit
    hash collides less than the literal low-bit remainder (reading R5)."""
    if which == "c2":  # g = 16: neighbour strides 16 and 256 are powers of two (R5)
        A, B, _ = synth.workload("c2_stencil64", scale=16)
    else:
        A, B, _ = synth.workload("c3_rmat20", scale=11)
    dA = spg.DeviceCSR.from_host(A)
    dB = dA if B is A else spg.DeviceCSR.from_host(B)
    st = spg.probe_stats(dA, dB, ctx=ctx)
    nnz = oracle.row_nnz(A, B)
    want_keys = int(nnz[(nnz > 0) & (2 * nnz <= 1024)].sum())
    _, f = oracle.flop(A, B)
    for mode, (probes, products, keys, c) in st.items():
        assert keys == want_keys, mode
        assert probes >= products > 0, mode
        assert products <= f
    if which == "c2":
        assert st["linear_high_bits"][3] < st["linear_low_bits"][3]


def test_c4_pruned_bitmask_growth(spg):
    """The pruning scatter's useful-entry bitmask is a grow-only workspace:
    a smaller A sizes it, a larger A must fall back to the full scan (and
    regrow), a repeat of the larger A uses the bitmask -- all exact."""
    ctx = spg.Context()
    for scale in (16, 17, 17, 16):  # nnz(A) 1.8 M / 3.6 M: both pruned
        A, B, _ = synth.workload("c4_tallskinny", scale=scale)
        assert A.nnz >= (1 << 20)
        gpu_vs_oracle(A, B, True, ctx=ctx, what=f"C4 s{scale} bitmask growth")


# ------------------------------------------------------------------ heap tier
def _heap_ctx(spg, mode):
    c = spg.Context()
    c.set_accumulator(mode)
    return c


def test_heap_tier_bitexact_c1(spg):
    """Heap SpGEMM on C1 with the heap forced for every eligible
    row: ascending columns by construction, and every entry summed in the
    oracle's canonical order with separate mul/add roundings -- BIT-exact."""
    A, B, _ = synth.workload("c1_er4096")
    ctx = _heap_ctx(spg, "heap")
    dA = spg.DeviceCSR.from_host(A)
    C = spg.spgemm(dA, dA, sorted=True, ctx=ctx)
    assert ctx.info()["heap_rows"] > 0.9 * A.nrows
    g_rp, g_col, g_val = C.to_host()
    o_rp, o_col, o_val = oracle.spgemm(A, B)
    assert np.array_equal(g_rp, o_rp) and np.array_equal(g_col, o_col)
    assert np.array_equal(g_val, o_val)  # bit-exact


def test_heap_auto_selector_cost_model(spg):
    """AUTO (with the paper's unit costs, h = 1) picks the heap exactly where
    Eq:heap_est < Eq:hash_est (c = 1.3) among the eligible rows (warp tiers, nnz(a_i) <= 16, flop_i <=
    2048, sorted B); C1 (low CR, short rows) goes mostly to the heap, C2's
    stencil's interior rows (nnz(a_i) = 27) are not eligible; results exact
    vs the oracle."""
    for name, want_some in (("c1_er4096", True), ("c2_stencil64", False)):
        A, B, _ = synth.workload(name, scale=None if name == "c1_er4096" else 16)
        ctx = spg.Context()
        ctx.set_accumulator("auto", 1.3, 1.0)
        gpu_vs_oracle(A, B, True, ctx=ctx, what=f"{name} auto")
        f, _ = oracle.flop(A, B)
        nz = oracle.row_nnz(A, B)
        na = np.diff(A.row_ptr)
        two_nz = np.maximum(2 * nz, 1)
        warp = (nz > 0) & (np.ceil(np.log2(two_nz)) <= 10) & ~((na > 512))
        elig = warp & (na <= 16) & (f <= 2048)
        th = f.astype(np.float32) * np.log2(np.maximum(na, 1).astype(np.float32))
        tc = f.astype(np.float32) * np.float32(1.3) + nz.astype(np.float32) * np.log2(
            np.maximum(nz, 1).astype(np.float32))
        pick = elig & (th < tc)
        near = elig & (np.abs(th - tc) <= 1e-5 * np.maximum(np.abs(tc), 1))
        got = ctx.info()["heap_rows"]
        assert abs(got - int(pick.sum())) <= int(near.sum()), (name, got, int(pick.sum()))
        if want_some:
            assert got > 0.5 * A.nrows


@pytest.mark.parametrize("seed", range(4))
def test_heap_tier_random_and_boundaries(spg, seed):
    """Forced heap on random shapes (empty rows, rectangular) and on rows at
    the eligibility edges (nnz(a_i) 16 / 17, flop 2048 / 2049): exact."""
    rng = np.random.default_rng(100 + seed)
    m, n, k = (int(x) for x in rng.integers(1, 400, size=3))
    A = synth.random_sparse(m, n, float(rng.uniform(0.005, 0.05)), seed, -1.0, 1.0, empty_rows=0.2)
    B = synth.random_sparse(n, k, float(rng.uniform(0.005, 0.1)), seed + 9, -1.0, 1.0, empty_rows=0.1)
    ctx = _heap_ctx(spg, "heap")
    g = spg.spgemm(spg.DeviceCSR.from_host(A), spg.DeviceCSR.from_host(B), sorted=True, ctx=ctx)
    o = oracle.spgemm(A, B)
    g_rp, g_col, g_val = g.to_host()
    assert np.array_equal(g_rp, o[0]) and np.array_equal(g_col, o[1])
    heap = ctx.info()["heap_rows"]
    assert heap > 0
    # heap rows are bit-exact, hashed rows within the signed-sum bound
    absA = synth.CSR(A.nrows, A.ncols, A.row_ptr, A.col, np.abs(A.val))
    absB = synth.CSR(B.nrows, B.ncols, B.row_ptr, B.col, np.abs(B.val))
    mag = oracle.spgemm(absA, absB)[2]
    assert (np.abs(g_val - o[2]) <= 1e-12 * mag).all()
    # eligibility edges
    specs = [(2048, 300), (2049, 300), (16 * 3, 16), (17 * 3, 17), (5, 5), (0, 0)]
    A2, B2 = synth.crafted_rows(specs, 5000, 40 + seed)
    gpu_vs_oracle(A2, B2, True, ctx=ctx, what="heap edges")


def test_heap_never_with_unsorted_b(spg):
    """The heap merge needs sorted B rows: with B's storage order shuffled
    the forced heap mode must fall back to hashing (and stay exact)."""
    A, B, _ = synth.workload("c1_er4096")
    Bs = synth.shuffle_within_rows(B, 3)
    ctx = _heap_ctx(spg, "heap")
    gpu_vs_oracle(A, Bs, True, ctx=ctx, what="heap, unsorted B")
    assert ctx.info()["heap_rows"] == 0
    ctx.set_accumulator("auto")
    gpu_vs_oracle(A, B, False, ctx=ctx, what="unsorted output: hash tiers")


def test_set_accumulator_errors(spg):
    from paper_1804_01698_b200 import _lib
    ctx = spg.Context()
    with pytest.raises(_lib.SpgError, match="INVALID_ARG"):
        _lib._check(ctx.handle, "x", _lib.load().spg_set_accumulator(ctx.handle, 7, 1.3, 8.0))
    with pytest.raises(_lib.SpgError, match="INVALID_ARG"):
        ctx.set_accumulator("auto", 1.3, 0.0)
    with pytest.raises(_lib.SpgError, match="INVALID_ARG"):
        ctx.set_accumulator("auto", 0.5)


# ------------------------------------------------------------------ one-phase
@pytest.mark.parametrize("sorted_out", [True, False])
def test_onephase_every_bin(spg, sorted_out):
    """One-phase multiply (tables sized by flop, no symbolic pass) on rows
    spanning every warp / block bin up to 8191 products (flop at T-1 / T /
    T+1 boundaries), shuffled and sorted B, plus C1 and a small C2: exact vs
    the oracle; rows beyond the block tier are refused (OVERFLOW)."""
    ctx = spg.Context()
    specs = []
    for h in [16, 32, 128, 256, 1024, 2048, 4096]:
        for f in (h - 1, h, h + 1):
            specs += [(f, max(1, f // 3)), (f, f)]
    specs += [(8191, 4000), (1, 1), (0, 0), (600, 2)]
    for shuffle in (False, True):
        A, B = synth.crafted_rows(specs, 1 << 16, 51, shuffle=shuffle)
        dA, dB = spg.DeviceCSR.from_host(A), spg.DeviceCSR.from_host(B)
        for rep in range(2):  # 1st call grows the workspace (rerun), 2nd is one round trip
            C = spg.spgemm(dA, dB, sorted=sorted_out, ctx=ctx, method="one_phase")
            compare(*C.to_host(), *oracle.spgemm(A, B), sorted_out, f"one-phase shuffle={shuffle}")
    for name, sc in (("c1_er4096", None), ("c2_stencil64", 12)):
        A, B, _ = synth.workload(name, scale=sc)
        dA = spg.DeviceCSR.from_host(A)
        C = spg.spgemm(dA, dA, sorted=sorted_out, ctx=ctx, method="one_phase")
        compare(*C.to_host(), *oracle.spgemm(A, B), sorted_out, f"one-phase {name}")
    A, B = synth.crafted_rows([(20000, 5000)], 1 << 16, 52)
    from paper_1804_01698_b200 import _lib
    with pytest.raises(_lib.SpgError, match="OVERFLOW"):
        spg.spgemm(spg.DeviceCSR.from_host(A), spg.DeviceCSR.from_host(B), ctx=ctx, method="one_phase")
    with pytest.raises(_lib.SpgError, match="STATE"):
        _lib.spg_onephase_emit(ctx.handle, 0, 0, 0)


def test_onephase_graph_replay(spg, monkeypatch):
    """The one-phase launch sequence is replayed as a CUDA graph when the
    inputs / workspace match the captured ones: repeated calls (and a call
    with new A values on the same structure) stay exact, and agree with a
    context that never captures (SPG_ONEPHASE_GRAPH=0)."""
    A, B, _ = synth.workload("c1_er4096")
    dA = spg.DeviceCSR.from_host(A)
    ctx = spg.Context()
    monkeypatch.setenv("SPG_ONEPHASE_GRAPH", "0")
    ctx0 = spg.Context()
    o = oracle.spgemm(A, B)
    for rep in range(3):
        C = spg.spgemm(dA, dA, sorted=True, ctx=ctx, method="one_phase")
        compare(*C.to_host(), *o, True, f"one-phase graph rep {rep}")
    l0 = ctx.launches
    C = spg.spgemm(dA, dA, sorted=True, ctx=ctx, method="one_phase")
    assert ctx.launches > l0  # replays count their kernels
    C0 = spg.spgemm(dA, dA, sorted=True, ctx=ctx0, method="one_phase")
    assert torch.equal(C.row_ptr, C0.row_ptr) and torch.equal(C.col, C0.col)
    # new values, same structure and buffers: the replayed graph reads them
    dA.val.copy_(torch.from_numpy(synth.with_values(A, 99, 0.5, 1.5).val).to(dA.val.device))
    A2 = synth.CSR(A.nrows, A.ncols, A.row_ptr, A.col, dA.val.cpu().numpy())
    C = spg.spgemm(dA, dA, sorted=True, ctx=ctx, method="one_phase")
    compare(*C.to_host(), *oracle.spgemm(A2, A2), True, "one-phase graph, new values")


@pytest.mark.parametrize("sorted_out", [True, False])
def test_column_parts_tile_records(spg, sorted_out):
    """Narrow hash parts index their columns by rank from the symbolic's tile
    records (bitmap words + ranks) once the ctx's record buffer is sized: the
    first multiply on a fresh ctx hashes (records not yet allocated), the
    second and third use the records -- all exact vs the oracle, and the
    records-off switch (SPG_TUNE bit 256) agrees."""
    specs = [(150000, 50000), (30000, 9000), (9000, 8193), (70000, 4097), (20000, 12000),
             (600000, 200000), (40000, 30000)]
    A, B = synth.crafted_rows(specs, 1_000_000, 17)
    dA, dB = spg.DeviceCSR.from_host(A), spg.DeviceCSR.from_host(B)
    o = oracle.spgemm(A, B)
    ctx = spg.Context()
    for rep in range(3):
        C = spg.spgemm(dA, dB, sorted=sorted_out, ctx=ctx)
        compare(*C.to_host(), *o, sorted_out, f"tile records rep {rep}")
    A3, B3, _ = synth.workload("c3_rmat20", scale=14)
    dA3 = spg.DeviceCSR.from_host(A3)
    o3 = oracle.spgemm(A3, B3)
    for rep in range(2):
        C = spg.spgemm(dA3, dA3, sorted=sorted_out, ctx=ctx)
        compare(*C.to_host(), *o3, sorted_out, f"C3 s14 tile records rep {rep}")


@pytest.mark.parametrize("sorted_out", [True, False])
def test_dense_window_negative_zero_products(spg, ctx, sorted_out):
    """Dense column windows mark absent slots with -0.0 (DESIGN.md reading
    R17): every product is mapped through v + (+0.0) first, so an entry whose
    only terms are -0.0 products (a_ik < 0 times b_kj = 0.0) is still present
    (structure is value-blind, reading R1) with value 0.0.  One long row with
    two heavy tiles (dense parts) and a multi-tile light run (hash part)."""
    A, B = _tile_rows([6000, 3000, 700, 0, 900], 8, 41)
    bval = B.val.copy()
    bval[B.row_ptr[2]:B.row_ptr[3]] = 0.0      # B row 2: every value +0.0
    bval[B.row_ptr[1]:B.row_ptr[2]] *= -1.0    # B row 1: negative values
    B = synth.CSR(B.nrows, B.ncols, B.row_ptr, B.col, bval)
    aval = A.val.copy()
    aval[2] = -1.25                            # a_02 < 0: -0.0 products
    A = synth.CSR(A.nrows, A.ncols, A.row_ptr, A.col, aval)
    o_rp, o_col, o_val = oracle.spgemm(A, B)
    assert (o_val == 0.0).sum() > 1000         # keys reached only through B row 2
    dA, dB = spg.DeviceCSR.from_host(A), spg.DeviceCSR.from_host(B)
    for rep in range(2):                       # (the second with tile records)
        C = spg.spgemm(dA, dB, sorted=sorted_out, ctx=ctx)
        compare(*C.to_host(), o_rp, o_col, o_val, sorted_out, f"-0.0 products rep {rep}")


@pytest.mark.parametrize("sorted_out", [True, False])
def test_block_tier_sorted_lists(spg, monkeypatch, sorted_out):
    """Sorted column lists (SPG_TUNE bit 65536, off by default): the bitmap
    symbolic writes each block-tier row's sorted columns and the numeric
    block tier accumulates by rank and emits by copying -- exact vs the
    oracle on R-MAT rows with 512 < nnz(c_i) <= 8192 (and the rows around
    them), twice on one ctx (the first call sizes the list buffer)."""
    monkeypatch.setenv("SPG_TUNE", "65536")
    ctx = spg.Context()
    A, B, _ = synth.workload("c3_rmat20", scale=15)
    dA = spg.DeviceCSR.from_host(A)
    o = oracle.spgemm(A, B)
    for rep in range(2):
        C = spg.spgemm(dA, dA, sorted=sorted_out, ctx=ctx)
        compare(*C.to_host(), *o, sorted_out, f"sorted lists rep {rep}")


def test_torch_allocator_callbacks(spg):
    """The C ABI's spg_alloc_fn / spg_free_fn (include/spgemm.h): a ctx whose
    workspace comes from the PyTorch caching allocator gives the oracle's
    result, grows through the callbacks (a second, larger product) and hands
    everything back on destroy."""
    ctx = spg.Context(allocator="torch")
    assert ctx.workspace_bytes == 0
    for n, seed in ((3000, 11), (40000, 12)):
        A = synth.er_poisson(n, 8.0, seed)
        for sorted_out in (True, False):
            gpu_vs_oracle(A, A, sorted_out, ctx=ctx, what=f"torch allocator n={n}")
        held = ctx.workspace_bytes
        assert held > 0 and len(ctx._live) > 0
    small = held
    A = synth.rmat(14, 16, seed=5)   # long rows: parts, tile offsets, slabs
    gpu_vs_oracle(A, A, True, ctx=ctx, what="torch allocator rmat14")
    assert ctx.workspace_bytes > small
    live = ctx._live
    del ctx
    import gc
    gc.collect()
    assert len(live) == 0
    with pytest.raises(ValueError):
        spg.Context(allocator="nope")
