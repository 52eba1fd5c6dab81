set -x
SPG_NVCC_EXTRA="-DSPG_TPART_INSTR=1" python -c "from paper_1804_01698_b200 import build; build.build(out='tools/ab_so/instr.so')" || exit 1
python - <<'PY' > gpurun_out/s3w_instr.log 2>&1
import os, sys
sys.path.insert(0, '.')
os.environ["SPG_SERIAL_BINS"] = "1"
from paper_1804_01698_b200 import _lib
_lib.load('tools/ab_so/instr.so')
import torch, synth, paper_1804_01698_b200 as spg
A, B, _ = synth.workload("c3_rmat20")
dA = spg.DeviceCSR.from_host(A)
for tune in ("0", "2048", "4096", "6144", "8192", "16"):
    os.environ["SPG_TUNE"] = tune
    ctx = spg.Context()
    for r in range(2):
        _lib.spg_profile_reset(ctx.handle); _lib.spg_profile_enable(ctx.handle, True)
        C = spg.spgemm(dA, dA, sorted=True, ctx=ctx); torch.cuda.synchronize(); del C
        _lib.spg_profile_enable(ctx.handle, False)
    rec = {n: round(t, 2) for n, t in _lib.spg_profile_records(ctx.handle) if n.startswith("k_num_tpart")}
    print("tune", tune, rec, "dbg", _lib.spg_debug_counters(ctx.handle), flush=True)
    del ctx
PY
