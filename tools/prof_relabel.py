"""Device time of the degree-ascending relabelling on C5's G:
CUDA events around spg.degree_relabel plus per-kernel records, and the
fused count on the result."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import synth  # noqa: E402
import paper_1804_01698_b200 as spg  # noqa: E402
from paper_1804_01698_b200 import _lib  # noqa: E402

L, U, ex = synth.workload("c5_triangle")
dG = spg.DeviceCSR.from_host(ex["G"])
ctx = spg.Context()
spg.degree_relabel(dG, ctx=ctx)
torch.cuda.synchronize()
for _ in range(3):
    a, b, c = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    _lib.spg_profile_reset(ctx.handle)
    _lib.spg_profile_enable(ctx.handle, True)
    a.record()
    _, L2, U2, G2 = spg.degree_relabel(dG, ctx=ctx)
    b.record()
    n = spg.triangle_count_fused(L2, U2, G2, ctx=ctx)
    c.record()
    torch.cuda.synchronize()
    _lib.spg_profile_enable(ctx.handle, False)
    recs = _lib.spg_profile_records(ctx.handle)
    print(f"relabel {a.elapsed_time(b):.3f} ms, fused count {b.elapsed_time(c):.3f} ms, triangles {n}",
          [(k, round(t, 3)) for k, t in recs if t > 0.05], flush=True)
