set -x
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "part or column or c3_rmat_small or bin_bound or wide or c5 or signed or records" > gpurun_out/r2_pytest18.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r2_pytest18.log
for so in 1 0; do SPG_TUNE=8 timeout 300 python tools/profile_step.py --config c3_rmat20 --records --reps 3 --sorted $so > gpurun_out/r2_prof18_c3_s$so.log 2>&1; done
python - <<'PY'
import ast
for f in ("gpurun_out/r2_prof18_c3_s1.log","gpurun_out/r2_prof18_c3_s0.log"):
    L=[l for l in open(f) if l.startswith("[(")]
    for l in L:
        d=dict((n,t) for n,t in ast.literal_eval(l))
        print(f.split('/')[-1], {k:v for k,v in d.items() if k in ('k_num_tpart<512>','k_sym_bitmap<1024>')})
    print([l for l in open(f) if l.startswith("dbg")][-1])
PY
