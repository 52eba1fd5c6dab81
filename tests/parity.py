"""Parity helpers: compare the CUDA path (through the C ABI) with the oracle.

Bar (BASELINE.json north_star):
  * row_ptr, per-row flop, table sizes: bit-exact (int64)
  * col_idx after a per-row sort of (col, val) pairs: bit-exact
  * with sorted=True: each GPU row strictly increasing BEFORE any re-sort
  * values: |g - o| <= 1e-12 |o| per entry (g == o when o == 0)
"""
from __future__ import annotations

import numpy as np

import oracle

RTOL = 1e-12


def sort_rows(rp, col, val):
    """Per-row sort of (col, val) pairs (for unsorted GPU output, reading R9)."""
    rows = np.repeat(np.arange(len(rp) - 1), np.diff(rp))
    order = np.lexsort((col, rows))
    return col[order], val[order]


def compare(g_rp, g_col, g_val, o_rp, o_col, o_val, sorted_out: bool, what=""):
    g_rp = np.asarray(g_rp) - g_rp[0]
    assert len(g_rp) == len(o_rp), what
    bad = np.nonzero(g_rp != o_rp)[0]
    assert len(bad) == 0, f"{what}: row_ptr differs at rows {bad[:10]}"
    if sorted_out:
        rows = np.repeat(np.arange(len(g_rp) - 1), np.diff(g_rp))
        d = np.diff(g_col.astype(np.int64))
        same_row = rows[1:] == rows[:-1]
        assert np.all(d[same_row] > 0), f"{what}: sorted output not strictly increasing"
    else:
        g_col, g_val = sort_rows(g_rp, g_col, g_val)
    assert np.array_equal(g_col, o_col), f"{what}: col_idx differs"
    err = np.abs(g_val - o_val)
    tol = RTOL * np.abs(o_val)
    viol = err > tol
    if viol.any():
        k = int(np.argmax(err / np.maximum(np.abs(o_val), 1e-300)))
        raise AssertionError(f"{what}: {int(viol.sum())} values outside 1e-12 rel; worst at {k}: "
                             f"gpu={g_val[k]!r} oracle={o_val[k]!r}")
    rel = err / np.maximum(np.abs(o_val), 1e-300)
    return float(rel.max()) if len(rel) else 0.0


def gpu_vs_oracle(A, B, sorted_out: bool, nthreads: int = 0, ctx=None, what=""):
    """Full comparison on the whole product (sizes the oracle finishes quickly)."""
    import paper_1804_01698_b200 as spg
    dA = spg.DeviceCSR.from_host(A)
    dB = dA if B is A else spg.DeviceCSR.from_host(B)
    C = spg.spgemm(dA, dB, sorted=sorted_out, ctx=ctx)
    g_rp, g_col, g_val = C.to_host()
    o_rp, o_col, o_val = oracle.spgemm(A, B, nthreads=nthreads)
    return compare(g_rp, g_col, g_val, o_rp, o_col, o_val, sorted_out, what)


def sampled_rows(A, B, flop_rows, nsample=200, seed=0, top=16):
    """Row ids for full-size sampled parity: heaviest rows, random non-empty rows,
    first and last rows."""
    rng = np.random.default_rng(seed)
    nz = np.nonzero(flop_rows)[0]
    heavy = np.argsort(flop_rows)[::-1][:top]
    rnd = rng.choice(nz, size=min(nsample, len(nz)), replace=False) if len(nz) else []
    ids = np.unique(np.r_[heavy, rnd, [0, A.nrows - 1]]).astype(np.int64)
    return ids


def compare_rows(C_dev, A, B, rows, sorted_out: bool, nthreads: int = 0, what=""):
    """Compare selected rows of a device C against the oracle row by row."""
    g_rp_all = C_dev.row_ptr.cpu().numpy()
    worst = 0.0
    for r in rows:
        r = int(r)
        s, e = int(g_rp_all[r]), int(g_rp_all[r + 1])
        g_col = C_dev.col[s:e].cpu().numpy()
        g_val = C_dev.val[s:e].cpu().numpy()
        o_rp, o_col, o_val = oracle.spgemm(A, B, r, r + 1, nthreads=nthreads)
        w = compare(np.array([0, e - s]), g_col, g_val, o_rp, o_col, o_val, sorted_out,
                    f"{what} row {r}")
        worst = max(worst, w)
    return worst
