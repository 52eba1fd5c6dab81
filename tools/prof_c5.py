"""Per-kernel breakdown of the config-5 triangle step (serialised bins)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["SPG_SERIAL_BINS"] = "1"
import torch  # noqa: E402
import synth  # noqa: E402
import paper_1804_01698_b200 as spg  # noqa: E402
from paper_1804_01698_b200 import _lib  # noqa: E402
L, U, ex = synth.workload("c5_triangle")
dL, dU, dG = (spg.DeviceCSR.from_host(x) for x in (L, U, ex["G"]))
ctx = spg.Context()
for sorted_out in (False, True):
    spg.triangle_count(dL, dU, dG, sorted=sorted_out, ctx=ctx)
    torch.cuda.synchronize()
    _lib.spg_profile_reset(ctx.handle)
    _lib.spg_profile_enable(ctx.handle, True)
    t0 = time.perf_counter()
    n = spg.triangle_count(dL, dU, dG, sorted=sorted_out, ctx=ctx)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    _lib.spg_profile_enable(ctx.handle, False)
    agg = {}
    for k, t in _lib.spg_profile_records(ctx.handle):
        agg[k] = agg.get(k, 0.0) + t
    print(f"sorted={sorted_out} triangles={n} wall={dt*1e3:.1f} ms kernels={sum(agg.values()):.1f} ms",
          sorted(((k, round(v, 1)) for k, v in agg.items()), key=lambda x: -x[1])[:10], flush=True)
t0 = time.perf_counter()
n2 = spg.triangle_count_fused(dL, dU, dG, ctx=ctx)
torch.cuda.synchronize()
print("fused", n2, (time.perf_counter() - t0) * 1e3, "ms")
