#!/bin/bash
cd "$(dirname "$0")/.."
F=numeric.cuh CFG=c2_stencil64 REPS=3 VS="old new old new" KPAT="k_num_warp<256>|k_sym_warp<1024>" bash tools/run_ab_src.sh > gpurun_out/ab_warp.log 2>&1
python -c "from paper_1804_01698_b200 import build; build.build(force=True)" > gpurun_out/build_new.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "c2 or c1 or warp or sorted or onephase or one_phase" > gpurun_out/ab_warp_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/ab_warp_tests.log
F=symbolic.cuh CFG=c3_rmat20 VS="old new old new" KPAT="k_sym_bitmap<1024>" bash tools/run_ab_src.sh > gpurun_out/ab_sym8.log 2>&1
