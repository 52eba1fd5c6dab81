set -x
python -c "from paper_1804_01698_b200 import build; build.build()" || exit 1
SPG_NVCC_EXTRA="-DSPG_TPART_INSTR=1" python -c "from paper_1804_01698_b200 import build; build.build(out='tools/ab_so/instr.so')" || exit 1
python - <<'PY' > gpurun_out/s3v_instr.log 2>&1
import os, sys
sys.path.insert(0, '.')
os.environ["SPG_SERIAL_BINS"] = "1"
from paper_1804_01698_b200 import _lib
_lib.load('tools/ab_so/instr.so')
import torch, synth, paper_1804_01698_b200 as spg
A, B, _ = synth.workload("c3_rmat20")
dA = spg.DeviceCSR.from_host(A)
ctx = spg.Context()
for r in range(2):
    C = spg.spgemm(dA, dA, sorted=True, ctx=ctx); torch.cuda.synchronize(); del C
    print("dbg", _lib.spg_debug_counters(ctx.handle))
for r in range(2):
    C = spg.spgemm(dA, dA, sorted=False, ctx=ctx); torch.cuda.synchronize(); del C
    print("dbg unsorted", _lib.spg_debug_counters(ctx.handle))
PY
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/s3v_bench_c3.json 2> gpurun_out/s3v_bench_c3.err; echo "bench rc=$?"
