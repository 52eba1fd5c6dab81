set -x
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "part or column or c3_rmat_small or bin_bound or wide" > gpurun_out/r2_pytest4.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r2_pytest4.log
SPG_TUNE=8 timeout 300 python tools/profile_step.py --config c3_rmat20 --records --reps 2 --sorted 1 > gpurun_out/r2_prof4_c3_s1.log 2>&1
grep -h "dbg" gpurun_out/r2_prof4_c3_s1.log | tail -1
timeout 300 python tools/profile_step.py --config c3_rmat20 --records --reps 2 --sorted 1 > gpurun_out/r2_prof4b_c3_s1.log 2>&1
timeout 300 python tools/profile_step.py --config c3_rmat20 --records --reps 2 --sorted 0 > gpurun_out/r2_prof4b_c3_s0.log 2>&1
python - <<'PY'
import ast
for f in ("gpurun_out/r2_prof4_c3_s1.log","gpurun_out/r2_prof4b_c3_s1.log","gpurun_out/r2_prof4b_c3_s0.log"):
    L=[l for l in open(f) if l.startswith("[(")]
    d=dict((n,t) for n,t in ast.literal_eval(L[-1]))
    print(f, {k:v for k,v in d.items() if v>1})
PY
