#!/bin/bash
# end-of-round evidence at HEAD: GPU tests, default bench (C3), its ncu launch list (one GPU)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
( time timeout 1500 python -m pytest tests -m gpu -x -q ) > gpurun_out/fin_pytest.log 2>&1
echo "pytest rc=$?" > gpurun_out/fin_rc.log
timeout 900 python bench.py > gpurun_out/fin_bench_c3.json 2> gpurun_out/fin_bench_c3.err
echo "bench rc=$?" >> gpurun_out/fin_rc.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/fin_launches_c3.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/fin_ncu_launch_c3.log 2>&1
echo "launch-list rc=$?" >> gpurun_out/fin_rc.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/fin_rc.log
