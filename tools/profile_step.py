"""Minimal driver for ncu: a few C = A*B calls on one workload (no oracle)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import synth  # noqa: E402
import paper_1804_01698_b200 as spg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2_stencil64")
ap.add_argument("--scale", type=int, default=None)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--sorted", type=int, default=1)
ap.add_argument("--records", action="store_true")
ap.add_argument("--rows", default=None, help="r0:r1 row-range view of A")
a = ap.parse_args()
A, B, _ = synth.workload(a.config, a.scale)
dA = spg.DeviceCSR.from_host(A)
dB = dA if B is A else spg.DeviceCSR.from_host(B)
if a.rows:
    r0, r1 = (int(x) for x in a.rows.split(":"))
    dA = dA.rows(r0, r1)
ctx = spg.Context()
from paper_1804_01698_b200 import _lib  # noqa: E402
for _ in range(a.reps):
    if a.records:
        _lib.spg_profile_reset(ctx.handle)
        _lib.spg_profile_enable(ctx.handle, True)
    C = spg.spgemm(dA, dB, sorted=bool(a.sorted), ctx=ctx)
    torch.cuda.synchronize()
    if a.records:
        _lib.spg_profile_enable(ctx.handle, False)
        print([(n, round(t, 3)) for n, t in _lib.spg_profile_records(ctx.handle)], flush=True)
        print(ctx.info(), flush=True)
        print("dbg", _lib.spg_debug_counters(ctx.handle), flush=True)
    del C
print("ok", ctx.info()["nnz_total"], ctx.launches)
