#!/bin/bash
cd "$(dirname "$0")/.."
FLAGS_A="" FLAGS_B="${FLAGS_B:--DSPG_ADD2=1}" bash tools/run_ab_flags.sh > gpurun_out/ab_add2.log 2>&1
SPG_NVCC_EXTRA="${FLAGS_B:--DSPG_ADD2=1}" python -c "from paper_1804_01698_b200 import build; build.build(force=True)" > gpurun_out/build_B.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "column or c3 or c5 or dense or signed" > gpurun_out/ab_add2_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/ab_add2_tests.log
