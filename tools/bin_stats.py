"""Per-tier statistics of one workload (measurement tool): rows, flop,
nnz(C) and the mean compression ratio of the numeric tiers (T_n = lowest 2^n
>= 2 nnz(c_i): warp <= 1024 slots, block 2K..16K, long rows nnz > 8192),
from one symbolic on the GPU (row_ptr of C, flop from the plan export).

    python tools/bin_stats.py --config c3_rmat20
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import synth  # noqa: E402
import paper_1804_01698_b200 as spg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3_rmat20")
ap.add_argument("--scale", type=int, default=None)
a = ap.parse_args()
A, B, _ = synth.workload(a.config, a.scale)
dA = spg.DeviceCSR.from_host(A)
dB = dA if B is A else spg.DeviceCSR.from_host(B)
ctx = spg.Context()
rp, nnz, flop = spg.spg_symbolic(dA, dB, ctx)
f, _ = spg.plan_export(ctx, A.nrows)
rn = (rp[1:] - rp[:-1]).double()
f = f.double()
na = torch.from_numpy(A.row_ptr[1:] - A.row_ptr[:-1]).to(f.device).double()
edges = [(0, 0, "empty"), (1, 128, "warp<256>"), (129, 512, "warp<1024>"), (513, 1024, "block 2K"),
         (1025, 2048, "block 4K"), (2049, 4096, "block 8K"), (4097, 8192, "block 16K"),
         (8193, 1 << 40, "long (parts)")]
print(f"{'tier':14s} {'rows':>9s} {'flop':>14s} {'nnz(C)':>14s} {'CR':>6s} {'flop/row':>9s} {'nnz(a)/row':>10s}")
for lo, hi, name in edges:
    m = (rn >= lo) & (rn <= hi)
    r = int(m.sum())
    fl, nz = float(f[m].sum()), float(rn[m].sum())
    print(f"{name:14s} {r:9d} {fl:14.0f} {nz:14.0f} {fl / max(nz, 1):6.2f} {fl / max(r, 1):9.0f} "
          f"{float(na[m].sum()) / max(r, 1):10.1f}")
print("total flop", flop, "nnz", nnz)
