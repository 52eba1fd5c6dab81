#!/usr/bin/env python
"""Write full-size oracle goldens for the BASELINE configs (test infrastructure).

Calls ONLY ``oracle/`` (and the seeded ``synth/`` generators); nothing here
touches the CUDA path, so every value it stores is the oracle's (task rule:
"a stored value is ... written by a committed script that calls only
oracle/").  Output: ``tests/golden/full_configs.json`` with, per config,

* flop total and nnz(C) (oracle_flop / oracle_symbolic);
* sha256 of the oracle's per-row nnz(c_i) as little-endian int64 (the GPU
  C.row_ptr differences must hash to the same value: an exact check of the
  structure of all rows without storing 8 MB per config);
* C5: the natural-order triangle count = sum(L*U o G) / 2 (Sec 5.6,
  P:602-605; BASELINE config 5), computed by oracle.triangle_count in row
  blocks.

Run: ``python tools/oracle_goldens.py [--configs c3_rmat20,c5_triangle,...]``
(minutes on 8 host cores; C5's count is the long one).
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import synth  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "full_configs.json")


def row_nnz_sha(nnz: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(nnz, dtype="<i8").tobytes()).hexdigest()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c1_er4096,c2_stencil64,c3_rmat20,c4_tallskinny,c5_triangle")
    args = ap.parse_args()
    data = {}
    if os.path.exists(OUT):
        data = json.load(open(OUT))
    data["_cite"] = ("Written by tools/oracle_goldens.py from oracle/ only (flop: P:252-259; "
                     "row nnz: symbolic P:285; triangles: Sec 5.6 P:602-605 with BASELINE "
                     "config 5's natural order, reading R13). row_nnz_sha256 = sha256 of the "
                     "per-row nnz(c_i) as little-endian int64.")
    for name in args.configs.split(","):
        t0 = time.time()
        A, B, extra = synth.workload(name)
        f, tot = oracle.flop(A, B)
        nnz = oracle.row_nnz(A, B)
        rec = {"m": A.nrows, "nnz_A": A.nnz, "nnz_B": B.nnz, "flop": int(tot),
               "nnz_C": int(nnz.sum()), "row_nnz_sha256": row_nnz_sha(nnz),
               "max_row_flop": int(f.max()) if len(f) else 0,
               "max_row_nnz": int(nnz.max()) if len(nnz) else 0}
        if name == "c5_triangle":
            G = extra["G"]
            rec["triangles"] = int(oracle.triangle_count(A, B, G, block_rows=1 << 15))
        rec["oracle_seconds"] = round(time.time() - t0, 1)
        data[name] = rec
        print(name, rec, flush=True)
        json.dump(data, open(OUT, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
