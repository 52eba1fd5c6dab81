set -x
python -c "from paper_1804_01698_b200 import build; build.build()" || exit 1
SPG_NVCC_EXTRA="-DSPG_SYM_INSTR=1" python -c "from paper_1804_01698_b200 import build; build.build(out='tools/ab_so/syminstr.so')" || exit 1
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/s3z_pytest.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/s3z_pytest.log
for r in 1 2; do
timeout 900 python tools/ab_tune.py --rounds 1 > gpurun_out/s3z_ab_new$r.log 2>&1
timeout 900 python tools/ab_tune.py --rounds 1 --so tools/ab_so/prev.so > gpurun_out/s3z_ab_prev$r.log 2>&1
done
grep -h tune= gpurun_out/s3z_ab_*.log
python - <<'PY' > gpurun_out/s3z_syminstr.log 2>&1
import os, sys
sys.path.insert(0, '.')
os.environ["SPG_SERIAL_BINS"] = "1"
from paper_1804_01698_b200 import _lib
_lib.load('tools/ab_so/syminstr.so')
import torch, synth, paper_1804_01698_b200 as spg
A, B, _ = synth.workload("c3_rmat20")
dA = spg.DeviceCSR.from_host(A)
ctx = spg.Context()
for r in range(2):
    rp, nnz, fl = spg.spg_symbolic(dA, dA, ctx); torch.cuda.synchronize()
    print("dbg", _lib.spg_debug_counters(ctx.handle), flush=True)
PY
cat gpurun_out/s3z_syminstr.log
