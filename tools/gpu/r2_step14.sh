set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "onephase" > gpurun_out/r2_pytest14.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r2_pytest14.log
for cfg in c1_er4096 c4_tallskinny; do timeout 900 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2_b14_$cfg.json 2> gpurun_out/r2_b14_$cfg.err; echo "bench $cfg rc=$?"; done
for cfg in c1_er4096 c4_tallskinny; do SPG_ONEPHASE_GRAPH=0 timeout 900 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-parity > gpurun_out/r2_b14_nograph_$cfg.json 2> gpurun_out/r2_b14_nograph_$cfg.err; echo "bench $cfg rc=$?"; done
