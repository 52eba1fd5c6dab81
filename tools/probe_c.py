"""Measured collision factor c (Eq:hash_est P:362) of the warp-tier numeric
tables on the full-size workloads (spg.probe_stats)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_1804_01698_b200 as spg  # noqa: E402

res = {}
for cfg in sys.argv[1:] or ["c2_stencil64", "c3_rmat20", "c1_er4096"]:
    A, B, _ = synth.workload(cfg)
    dA = spg.DeviceCSR.from_host(A)
    dB = dA if B is A else spg.DeviceCSR.from_host(B)
    st = spg.probe_stats(dA, dB)
    res[cfg] = {m: {"probes": p, "products": n, "keys": k, "c": round(c, 4)} for m, (p, n, k, c) in st.items()}
    print(cfg, {m: v["c"] for m, v in res[cfg].items()}, "products", st["linear_high_bits"][1], flush=True)
print(json.dumps(res))
