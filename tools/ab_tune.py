"""In-process A/B of SPG_TUNE variants: the workload is generated once, then
for each round of variants (A, B, A, B, ...) a fresh ctx is created with the
variant's SPG_TUNE, warmed (records grown) and timed per kernel from the
ctx's profile records (serialised bins).  Prints one line per (variant,
round) with the chosen kernels' times and the step's kernel-time sum.

    python tools/ab_tune.py --config c3_rmat20 --tunes 0,512 --rounds 2
"""
import argparse
import gc
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import synth  # noqa: E402
import paper_1804_01698_b200 as spg  # noqa: E402
from paper_1804_01698_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3_rmat20")
ap.add_argument("--scale", type=int, default=None)
ap.add_argument("--tunes", default="0")
ap.add_argument("--rounds", type=int, default=2)
ap.add_argument("--sorted", type=int, default=1)
ap.add_argument("--kernels", default="k_num_tpart,k_sym_bitmap")
ap.add_argument("--so", default=None, help="library variant to load (A/B builds)")
a = ap.parse_args()
if a.so:
    _lib.load(a.so)
os.environ["SPG_SERIAL_BINS"] = "1"
A, B, _ = synth.workload(a.config, a.scale)
dA = spg.DeviceCSR.from_host(A)
dB = dA if B is A else spg.DeviceCSR.from_host(B)
pats = a.kernels.split(",")
for rnd in range(a.rounds):
    for t in a.tunes.split(","):
        os.environ["SPG_TUNE"] = t
        ctx = spg.Context()
        for rep in range(2):  # warm-up (records sized) + timed
            _lib.spg_profile_reset(ctx.handle)
            _lib.spg_profile_enable(ctx.handle, True)
            C = spg.spgemm(dA, dB, sorted=bool(a.sorted), ctx=ctx)
            torch.cuda.synchronize()
            _lib.spg_profile_enable(ctx.handle, False)
            recs = _lib.spg_profile_records(ctx.handle)
            del C
        tot = sum(ms for _, ms in recs)
        sel = {p: round(sum(ms for n, ms in recs if n.startswith(p)), 3) for p in pats}
        print(f"so={a.so} tune={t} round={rnd} {sel} step_kernels={tot:.3f}", flush=True)
        del ctx
        gc.collect()
        torch.cuda.empty_cache()
