#!/bin/bash
# last confirmation at the final HEAD: GPU suite, smoke, default bench (C3) + its ncu launch list, C5 line
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
( time timeout 1500 python -m pytest tests -m gpu -x -q ) > gpurun_out/fin5_pytest.log 2>&1
echo "pytest rc=$?" > gpurun_out/fin5_rc.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin5_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/fin5_rc.log
timeout 900 python bench.py > gpurun_out/fin5_bench_c3_rmat20.json 2> gpurun_out/fin5_bench_c3_rmat20.err
echo "c3 rc=$?" >> gpurun_out/fin5_rc.log
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/fin5_reference_c3.json 2> gpurun_out/fin5_reference_c3.err
echo "reference rc=$?" >> gpurun_out/fin5_rc.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/fin5_launches_c3.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/fin5_ncu_launch_c3.log 2>&1
echo "launch-list rc=$?" >> gpurun_out/fin5_rc.log
timeout 1200 python bench.py --config c5_triangle --steps 3 > gpurun_out/fin5_bench_c5_triangle.json 2> gpurun_out/fin5_bench_c5_triangle.err
echo "c5 rc=$?" >> gpurun_out/fin5_rc.log
