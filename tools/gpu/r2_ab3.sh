for rep in 1 2; do
for v in base d4 d8; do
  cp tools/ab_so/libspgemm_$v.so paper_1804_01698_b200/libspgemm.so; touch paper_1804_01698_b200/libspgemm.so
  for cfg in c2_stencil64 c3_rmat20; do
    timeout 300 python tools/profile_step.py --config $cfg --records --reps 4 --sorted 1 > gpurun_out/ab3_${v}_$cfg.log 2>&1
    python - "$v" "$cfg" <<'PY'
import ast,sys
L=[l for l in open(f"gpurun_out/ab3_{sys.argv[1]}_{sys.argv[2]}.log") if l.startswith("[(")]
tot={}
for l in L[2:]:
    for n,t in ast.literal_eval(l): tot[n]=tot.get(n,0)+t/len(L[2:])
print(sys.argv[1], sys.argv[2], {k:round(v,3) for k,v in tot.items() if v>0.02}, flush=True)
PY
  done
done
done
