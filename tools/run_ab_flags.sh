#!/bin/bash
# A/B of nvcc define sets (FLAGS_A / FLAGS_B) on one config
cd "$(dirname "$0")/.."
for v in A B A B; do
  if [ $v = A ]; then fl="$FLAGS_A"; else fl="$FLAGS_B"; fi
  SPG_NVCC_EXTRA="$fl" python -c "from paper_1804_01698_b200 import build; build.build(force=True)" > gpurun_out/build_$v.log 2>&1 || exit 1
  SPG_SERIAL_BINS=1 timeout 600 python tools/profile_step.py --config ${CFG:-c3_rmat20} --reps 2 --sorted ${SO:-1} --records \
      > gpurun_out/abf_${v}.log 2>&1
  echo "$v: $(grep -oE "\((${KPAT:-.k_num_tpart<512>.|.k_sym_bitmap<1024>.}), [0-9.]*\)" gpurun_out/abf_${v}.log | tr '\n' ' ') $(tail -1 gpurun_out/abf_${v}.log)"
done
