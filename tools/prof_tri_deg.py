"""Triangle count on the degree-ordered split: relabel (untimed), then
the fused mask-and-sum; per-kernel records (one stream)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import synth  # noqa: E402
import paper_1804_01698_b200 as spg  # noqa: E402
from paper_1804_01698_b200 import _lib  # noqa: E402
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
L, U, ex = synth.workload("c5_triangle")
dG = spg.DeviceCSR.from_host(ex["G"])
ctx = spg.Context()
_, L2, U2, G2 = spg.degree_relabel(dG, ctx=ctx)
spg.triangle_count_fused(L2, U2, G2, ctx=ctx)
torch.cuda.synchronize()
for _ in range(reps):
    _lib.spg_profile_reset(ctx.handle)
    _lib.spg_profile_enable(ctx.handle, True)
    t0 = time.perf_counter()
    n = spg.triangle_count_fused(L2, U2, G2, ctx=ctx)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    _lib.spg_profile_enable(ctx.handle, False)
    print(f"triangles={n} wall={dt*1e3:.2f} ms", _lib.spg_profile_records(ctx.handle), flush=True)
