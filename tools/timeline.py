"""Diagnose a step: host-side phase timestamps + device events + per-launch records."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
import paper_1804_01698_b200 as spg  # noqa: E402
from paper_1804_01698_b200 import _lib  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2_stencil64"
A, B, _ = synth.workload(cfg)
dA = spg.DeviceCSR.from_host(A)
dB = dA if B is A else spg.DeviceCSR.from_host(B)
ctx = spg.Context()
flush = torch.empty(64 << 20, dtype=torch.int32, device="cuda")
for so in (True, False, True, False):
    for prof in (False, True):
        for it in range(3):
            flush.fill_(it)
            torch.cuda.synchronize()
            if prof:
                _lib.spg_profile_reset(ctx.handle)
                _lib.spg_profile_enable(ctx.handle, True)
            e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            t0 = time.perf_counter()
            e0.record()
            rp, nnz, _ = spg.spg_symbolic(dA, dB, ctx)
            t1 = time.perf_counter()
            e1.record()
            C = spg.spg_numeric(dA, dB, rp, nnz, so, ctx)
            t2 = time.perf_counter()
            e2.record()
            torch.cuda.synchronize()
            t3 = time.perf_counter()
            recs = []
            if prof:
                _lib.spg_profile_enable(ctx.handle, False)
                recs = _lib.spg_profile_records(ctx.handle)
            print(f"sorted={so} prof={prof} it={it}: host sym {1e3*(t1-t0):.3f} num-launch {1e3*(t2-t1):.3f} "
                  f"sync {1e3*(t3-t2):.3f} | dev sym {e0.elapsed_time(e1):.3f} num {e1.elapsed_time(e2):.3f} ms",
                  flush=True)
            if prof and it == 2:
                print("   ", [(n, round(t, 3)) for n, t in recs], flush=True)
            del C, rp
