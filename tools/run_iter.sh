#!/bin/bash
# one build-measure iteration on the GPU box.  env: TESTS=1 C2=1 C3PROF=1 UB=1 NCU=<kernel regex> NCUCFG=<config> NCUARGS
cd "$(dirname "$0")/.."
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo "build failed"; exit 1; }
if [ -n "$TESTS" ]; then timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log; fi
if [ -n "$C2" ]; then timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; fi
if [ -n "$C3PROF" ]; then CFGS="${C3PROF_CFGS:-c3_rmat20}" bash tools/run_prof_big.sh; fi
if [ -n "$UB" ]; then timeout 300 ./tools/ubench_dsmem > gpurun_out/ubench_dsmem.log 2>&1; fi
if [ -n "$NCU" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$NCU" -c ${NCUC:-1} \
    -o gpurun_out/full_iter -f python tools/profile_step.py --config ${NCUCFG:-c2_stencil64} ${NCUARGS} > gpurun_out/ncu_iter.log 2>&1
fi
