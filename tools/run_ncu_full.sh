#!/bin/bash
# ncu --set full captures of the top kernels (C2 warp tiers; C3 heavy-row tiers)
cd "$(dirname "$0")/.."
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_num_warp|k_sym_warp" -s 2 -c 2 \
    -o gpurun_out/full_c2 -f python tools/profile_step.py --reps 2 > gpurun_out/ncu_full_c2.log 2>&1
echo "c2 rc=$?" >> gpurun_out/ncu_full.log
SPG_SERIAL_BINS=1 ncu --set full --clock-control none --import-source on -k regex:"k_num_part|k_num_wpart|k_sym_bitmap" -c 3 \
    -o gpurun_out/full_c3 -f python tools/profile_step.py --config c3_rmat20 --reps 1 --sorted 0 > gpurun_out/ncu_full_c3.log 2>&1
echo "c3 rc=$?" >> gpurun_out/ncu_full.log
