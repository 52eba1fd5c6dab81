#!/usr/bin/env python
"""Full-size, ALL-rows parity of C3 (and C2 / C4) against the oracle, streamed
in row blocks (SURVEY.md §8(c) parity protocol item 5).  Too slow for the
pytest suite (C3's C has 9.7e9 entries, 116 GB); run once on the GPU box:

    python tools/parity_full.py [--config c3_rmat20] [--sorted 1] [--block-entries N]

For every block of rows [r0, r1): the GPU block of the last C (sorted) is
copied to the host and compared with oracle.spgemm(A, B, r0, r1): row_ptr
exact, columns exact (strictly increasing), values within 1e-12 relative.
Unsorted output: rows are re-sorted per row before the column comparison.
Prints one JSON line with the totals (kept under profiles/)."""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracle  # noqa: E402
import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3_rmat20")
    ap.add_argument("--sorted", type=int, default=1)
    ap.add_argument("--block-entries", type=int, default=1 << 28)
    ap.add_argument("--row-start", type=int, default=0, help="resume: compare rows [row-start, m) only")
    args = ap.parse_args()
    import torch
    import paper_1804_01698_b200 as spg
    from parity import sort_rows

    t0 = time.time()
    A, B, _ = synth.workload(args.config)
    dA = spg.DeviceCSR.from_host(A)
    dB = dA if B is A else spg.DeviceCSR.from_host(B)
    C = spg.spgemm(dA, dB, sorted=bool(args.sorted))
    torch.cuda.synchronize()
    g_rp = C.row_ptr.cpu().numpy()
    nnz = int(g_rp[-1])
    rows_done = ents = 0
    worst = 0.0
    bad_struct = bad_vals = 0
    r0 = args.row_start
    t_oracle = 0.0
    while r0 < A.nrows:
        r1 = int(np.searchsorted(g_rp, g_rp[r0] + args.block_entries, side="right")) - 1
        r1 = min(max(r1, r0 + 1), A.nrows)
        to = time.time()
        o_rp, o_col, o_val = oracle.spgemm(A, B, r0, r1)
        t_oracle += time.time() - to
        s, e = int(g_rp[r0]), int(g_rp[r1])
        grp = g_rp[r0:r1 + 1] - s
        gc = C.col[s:e].cpu().numpy()
        gv = C.val[s:e].cpu().numpy()
        if not np.array_equal(grp, o_rp):
            bad_struct += int((grp != o_rp).sum())
        else:
            if args.sorted:
                rows = np.repeat(np.arange(r1 - r0), np.diff(grp))
                d = np.diff(gc.astype(np.int64))
                bad_struct += int((d[rows[1:] == rows[:-1]] <= 0).sum())
            else:
                gc, gv = sort_rows(grp, gc, gv)
            if not np.array_equal(gc, o_col):
                bad_struct += int((gc != o_col).sum())
            else:
                rel = np.abs(gv - o_val) / np.maximum(np.abs(o_val), 1e-300)
                bad_vals += int((rel > 1e-12).sum())
                if len(rel):
                    worst = max(worst, float(rel.max()))
        rows_done += r1 - r0
        ents += e - s
        print(f"rows [{r0}, {r1}) entries {e - s} worst so far {worst:.3e}", file=sys.stderr, flush=True)
        r0 = r1
    out = {"config": args.config, "sorted": bool(args.sorted), "rows_checked": rows_done,
           "rows_total": A.nrows, "entries_checked": ents, "nnz_C": nnz, "structure_mismatches": bad_struct,
           "value_violations": bad_vals, "max_rel_err": worst, "tolerance": 1e-12,
           "row_start": args.row_start,
           "ok": bad_struct == 0 and bad_vals == 0 and ents == nnz - int(g_rp[args.row_start]),
           "oracle_seconds": round(t_oracle, 1), "wall_seconds": round(time.time() - t0, 1),
           "oracle_threads": os.cpu_count()}
    print(json.dumps(out), flush=True)
    return 0 if out["ok"] else 1


if __name__ == "__main__":
    sys.exit(main())
