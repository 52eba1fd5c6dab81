set -x
python -c "from paper_1804_01698_b200 import build; build.build()" || exit 1
SPG_NVCC_EXTRA="-DSPG_TPART_INSTR=1" python -c "from paper_1804_01698_b200 import build; build.build(out='tools/ab_so/instr.so')" || exit 1
timeout 900 python tools/ab_tune.py --rounds 1 --so tools/ab_so/instr.so > gpurun_out/s3t_instr.log 2>&1
python - <<'PY' >> gpurun_out/s3t_instr.log 2>&1
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
PY
mkdir -p gpurun_out/s3
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"k_num_tpart|k_sym_bitmap" --launch-skip 2 -c 2 -o gpurun_out/s3/c3s19c python tools/profile_step.py --config c3_rmat20 --scale 19 --reps 2 --sorted 1 > gpurun_out/s3/ncu19c.log 2>&1; echo "ncu rc=$?"
