#!/bin/bash
# phase clocks of the parts kernel / bitmap symbolic (instrumented build), then
# an ncu --set full capture of the current C3 top kernels (product build)
cd "$(dirname "$0")/.."
SPG_NVCC_EXTRA="-DSPG_TPART_INSTR=1" python -c "from paper_1804_01698_b200 import build; build.build(force=True)" > gpurun_out/build_instr.log 2>&1 || exit 1
SPG_SERIAL_BINS=1 timeout 600 python tools/profile_step.py --config c3_rmat20 --reps 2 --sorted 1 --records > gpurun_out/phase_c3.log 2>&1
echo "phase rc=$?" >> gpurun_out/phase_c3.log
python -c "from paper_1804_01698_b200 import build; build.build(force=True)" > gpurun_out/build.log 2>&1 || exit 1
SPG_SERIAL_BINS=1 timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_num_tpart|k_sym_bitmap|k_num_block" -c 4 \
    -o gpurun_out/r02f_c3 -f python tools/profile_step.py --config c3_rmat20 --reps 1 --sorted 1 > gpurun_out/r02f_ncu_c3.log 2>&1
echo "ncu rc=$?" >> gpurun_out/r02f_ncu_c3.log
