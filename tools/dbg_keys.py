import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch, synth, oracle
import paper_1804_01698_b200 as spg
specs = [(150000, 50000), (30000, 9000), (9000, 8193), (8193, 8193), (70000, 4097),
         (20000, 12000), (5, 5), (0, 0), (600000, 200000)]
A, B = synth.crafted_rows(specs, 1_000_000, 14)
dA, dB = spg.DeviceCSR.from_host(A), spg.DeviceCSR.from_host(B)
ctx = spg.Context()
o_rp, o_col, o_val = oracle.spgemm(A, B)
for rep in range(2):
    C = spg.spgemm(dA, dB, sorted=True, ctx=ctx)
    rp, col, val = C.to_host()
    for i in range(A.nrows):
        s, e = rp[i], rp[i+1]
        c = col[s:e].astype(np.int64)
        oc = o_col[o_rp[i]:o_rp[i+1]]
        bad = np.nonzero(np.diff(c) <= 0)[0]
        if len(bad) or not np.array_equal(c, oc):
            print(f"rep {rep} row {i}: nnz {e-s}, first bad {bad[:5]}, around {c[max(0,bad[0]-3):bad[0]+4] if len(bad) else None}, equal_as_set {np.array_equal(np.sort(c), oc)}", flush=True)
            if len(bad):
                b = bad[0]
                print("  tile of bad", c[b] >> 13, c[b+1] >> 13, "first mismatch idx", np.nonzero(c != oc)[0][:3] if len(c)==len(oc) else None)
    print("rep", rep, "done", flush=True)
