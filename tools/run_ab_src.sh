#!/bin/bash
# A/B of two versions of one source file (tools/_old_<f>, tools/_new_<f>) on one config
cd "$(dirname "$0")/.."
F=${F:-symbolic.cuh}
for v in ${VS:-old new old new}; do
  cp tools/_${v}_$F paper_1804_01698_b200/csrc/$F
  python -c "from paper_1804_01698_b200 import build; build.build(force=True)" > gpurun_out/build_$v.log 2>&1 || exit 1
  SPG_SERIAL_BINS=1 timeout 600 python tools/profile_step.py --config ${CFG:-c2_stencil64} --reps ${REPS:-2} --sorted ${SO:-1} --records \
      > gpurun_out/absrc_${v}.log 2>&1
  echo "$v: $(grep -oE "\('(${KPAT:-k_num_warp<256>|k_sym_warp<1024>|k_num_tpart<512>|k_sym_bitmap<1024>})', [0-9.]*\)" gpurun_out/absrc_${v}.log | tr '\n' ' ')"
done
cp tools/_new_$F paper_1804_01698_b200/csrc/$F
