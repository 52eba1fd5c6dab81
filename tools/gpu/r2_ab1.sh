# A/B of prebuilt variants (tools/ab_so/libspgemm_<v>.so) on C3
for rep in 1 2; do
for v in base ls8 ls32; do
  cp tools/ab_so/libspgemm_$v.so paper_1804_01698_b200/libspgemm.so; touch paper_1804_01698_b200/libspgemm.so
  for so in 1 0; do
    timeout 300 python tools/profile_step.py --config c3_rmat20 --records --reps 2 --sorted $so > gpurun_out/ab1_${v}_s$so.log 2>&1
    python - "$v" "$so" <<'PY'
import ast,sys
L=[l for l in open(f"gpurun_out/ab1_{sys.argv[1]}_s{sys.argv[2]}.log") if l.startswith("[(")]
d=dict((n,t) for n,t in ast.literal_eval(L[-1]))
print(sys.argv[1], "sorted" if sys.argv[2]=="1" else "unsorted", "tpart", d.get("k_num_tpart<512>"), "symbm", d.get("k_sym_bitmap<1024>"), flush=True)
PY
  done
done
done
