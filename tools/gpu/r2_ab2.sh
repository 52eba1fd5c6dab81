# phase costs of the parts kernel on C3 (SPG_TUNE 16: no emit; 32: no accumulation and no emit)
for t in 0 16 32; do
  for so in 1 0; do
    SPG_TUNE=$t timeout 300 python tools/profile_step.py --config c3_rmat20 --records --reps 2 --sorted $so > gpurun_out/ab2_t${t}_s$so.log 2>&1
    python - "$t" "$so" <<'PY'
import ast,sys
L=[l for l in open(f"gpurun_out/ab2_t{sys.argv[1]}_s{sys.argv[2]}.log") if l.startswith("[(")]
d=dict((n,t) for n,t in ast.literal_eval(L[-1]))
print("tune", sys.argv[1], "sorted" if sys.argv[2]=="1" else "unsorted", "tpart", d.get("k_num_tpart<512>"), flush=True)
PY
  done
done
