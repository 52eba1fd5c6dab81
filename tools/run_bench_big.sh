#!/bin/bash
# bench lines of the large configs (one GPU)
for cfg in c4_tallskinny c3_rmat20 c5_triangle c1_er4096; do
  timeout 900 python bench.py --config $cfg --steps 3 --warmup 3 --e2e-steps 1 --cpu-seconds 8 \
     > gpurun_out/bench_$cfg.json 2> gpurun_out/bench_$cfg.err
  echo "$cfg rc=$?" >> gpurun_out/bench_big.log
done
