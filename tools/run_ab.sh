#!/bin/bash
# A/B of SPG_TUNE variants on one config (serialised bins, profile records)
cd "$(dirname "$0")/.."
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
for t in ${TUNES:-0 1 2 3}; do
  for so in ${SORTS:-0}; do
    SPG_TUNE=$t SPG_SERIAL_BINS=1 timeout 600 python tools/profile_step.py --config ${CFG:-c3_rmat20} ${ARGS} --reps 2 --sorted $so --records \
      > gpurun_out/ab_t${t}_s${so}.log 2>&1
  done
done
