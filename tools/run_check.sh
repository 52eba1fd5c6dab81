#!/bin/bash
# GPU tests + default bench + big-config bench lines (one GPU)
cd "$(dirname "$0")/.."
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
echo "bench rc=$?" >> gpurun_out/bench_c2.err
for cfg in ${BIG_CFGS:-c4_tallskinny c3_rmat20 c5_triangle c1_er4096}; do
  timeout 900 python bench.py --config $cfg --steps 3 --warmup 3 --e2e-steps 1 --cpu-seconds 8 \
     > gpurun_out/bench_$cfg.json 2> gpurun_out/bench_$cfg.err
  echo "$cfg rc=$?" >> gpurun_out/bench_big.log
done
