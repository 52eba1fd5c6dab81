"""Parity soak (not part of the suite): many seeded random shapes, R-MAT
scales and skewed crafted rows through the CUDA path vs the oracle, both
output orders.  Usage: python tools/soak.py [n_seeds]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np  # noqa: E402
import synth  # noqa: E402
import paper_1804_01698_b200 as spg  # noqa: E402
from parity import gpu_vs_oracle  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100
ctx = spg.Context()
bad = 0
for seed in range(n):
    rng = np.random.default_rng(1000 + seed)
    kind = seed % 4
    if kind == 0:   # random shapes, some long rows
        m, nn, k = (int(x) for x in rng.integers(1, 3000, size=3))
        A = synth.random_sparse(m, nn, float(rng.uniform(0.0005, 0.05)), seed, 0.0, 1.0, empty_rows=0.2)
        B = synth.random_sparse(nn, k, float(rng.uniform(0.0005, 0.2)), seed + 7, 0.0, 1.0, empty_rows=0.1)
    elif kind == 1:  # R-MAT A^2 (hub B rows, column parts)
        A = synth.rmat(int(rng.integers(9, 14)), 16, seed)
        B = A
    elif kind == 2:  # R-MAT with shuffled storage order (unsorted inputs)
        A = synth.shuffle_within_rows(synth.rmat(int(rng.integers(9, 13)), 8, seed), seed)
        B = A
    else:            # one dense-ish B row hit by many a_ik (long-row deferral)
        nn = int(rng.integers(100, 2000))
        A = synth.random_sparse(int(rng.integers(10, 500)), nn, 0.2, seed, 0.0, 1.0)
        B = synth.random_sparse(nn, int(rng.integers(1000, 200000)), 0.002, seed + 3, 0.0, 1.0)
    for so in (True, False):
        try:
            gpu_vs_oracle(A, B, so, ctx=ctx, what=f"soak{seed}/{kind}/{so}")
        except AssertionError as e:
            bad += 1
            print("FAIL", seed, kind, so, str(e)[:200], flush=True)
    if seed % 10 == 9:
        print("done", seed + 1, "fails", bad, flush=True)
# triangle counting on random graphs: natural order (C formed and fused) and
# the degree relabelling, against the oracle's count
import oracle  # noqa: E402
tbad = 0
for seed in range(max(1, n // 4)):
    rng = np.random.default_rng(5000 + seed)
    G = synth.symmetrise_pattern(synth.rmat(int(rng.integers(8, 12)), int(rng.integers(4, 16)), seed),
                                 drop_diagonal=True)
    L, U = synth.tril_strict(G), synth.triu_strict(G)
    want = oracle.triangle_count(L, U, G)
    dL, dU, dG = (spg.DeviceCSR.from_host(x) for x in (L, U, G))
    got = (spg.triangle_count(dL, dU, dG, sorted=bool(seed % 2), ctx=ctx),
           spg.triangle_count_fused(dL, dU, dG, ctx=ctx), spg.triangle_count_graph(dG, ctx=ctx))
    if any(g != want for g in got):
        tbad += 1
        print("TRI FAIL", seed, want, got, flush=True)
print("soak", n, "cases x2 orders, failures:", bad, "; triangle graphs", max(1, n // 4),
      "failures:", tbad)
bad += tbad
sys.exit(1 if bad else 0)
