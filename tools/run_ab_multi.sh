#!/bin/bash
# A/B of several nvcc define sets on one config: FLAGSETS="set0|set1|set2" (| separated), ROUNDS repeats
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
IFS='|' read -ra SETS <<< "${FLAGSETS:-}"
for rnd in $(seq 1 ${ROUNDS:-2}); do
  for i in "${!SETS[@]}"; do
    fl="${SETS[$i]}"
    SPG_NVCC_EXTRA="$fl" python -c "from paper_1804_01698_b200 import build; build.build(force=True)" > gpurun_out/build_v$i.log 2>&1 || { echo "build $i failed"; exit 1; }
    SPG_SERIAL_BINS=1 timeout 600 python tools/profile_step.py --config ${CFG:-c2_stencil64} --reps 3 --sorted ${SO:-1} --records \
        > gpurun_out/abm_v${i}_r$rnd.log 2>&1
    echo "set$i [$fl] round $rnd: $(grep -oE "\((${KPAT:-.k_num_warp<256>.|.k_sym_warp<1024>.}), [0-9.]*\)" gpurun_out/abm_v${i}_r$rnd.log | tr '\n' ' ')"
  done
done
# leave the product build in place
python -c "from paper_1804_01698_b200 import build; build.build(force=True)" > gpurun_out/build_final.log 2>&1
