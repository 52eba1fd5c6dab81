#!/bin/bash
# serialised per-kernel breakdown of the big configs (profile records, bins on one stream)
cd "$(dirname "$0")/.."
for cfg in ${CFGS:-c3_rmat20 c5_triangle}; do
  for so in 1 0; do
    SPG_SERIAL_BINS=1 timeout 900 python tools/profile_step.py --config $cfg --reps 2 --sorted $so --records \
      > gpurun_out/prof_${cfg}_s$so.log 2>&1
  done
done
