#!/bin/bash
cd "$(dirname "$0")/.."
F=symbolic.cuh CFG=c3_rmat20 VS="old new old new" bash tools/run_ab_src.sh > gpurun_out/ab_sym.log 2>&1
python -c "from paper_1804_01698_b200 import build; build.build(force=True)" > gpurun_out/build_new.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "column or c3 or c5 or bitmap or wide or tier" > gpurun_out/ab_sym_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/ab_sym_tests.log
