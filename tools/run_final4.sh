#!/bin/bash
# end-of-round check after the CAS-first probing defaults and the barrier-free flop pass: suite, bench lines, ncu of the C2 warp tiers
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
( time timeout 1500 python -m pytest tests -m gpu -x -q ) > gpurun_out/fin4_pytest.log 2>&1
echo "pytest rc=$?" > gpurun_out/fin4_rc.log
for cfg in c2_stencil64 c4_tallskinny c1_er4096; do
  timeout 900 python bench.py --config $cfg > gpurun_out/fin4_bench_$cfg.json 2> gpurun_out/fin4_bench_$cfg.err
  echo "$cfg rc=$?" >> gpurun_out/fin4_rc.log
done
timeout 900 python bench.py > gpurun_out/fin4_bench_c3_rmat20.json 2> gpurun_out/fin4_bench_c3_rmat20.err
echo "c3 rc=$?" >> gpurun_out/fin4_rc.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_num_warp|k_sym_warp" -c 6 \
    -o gpurun_out/fin4_full_c2 -f python tools/profile_step.py --reps 2 > gpurun_out/fin4_ncu_full_c2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_flop_nz" -s 1 -c 1 \
    -o gpurun_out/fin4_full_c4 -f python tools/profile_step.py --config c4_tallskinny --reps 2 --sorted 0 > gpurun_out/fin4_ncu_full_c4.log 2>&1
python tools/ncu_summary.py gpurun_out/fin4_ncu_summary.md C2=gpurun_out/fin4_full_c2.ncu-rep C4=gpurun_out/fin4_full_c4.ncu-rep > /dev/null 2>&1
timeout 600 python tools/soak.py 100 > gpurun_out/fin4_soak.log 2>&1
echo "soak rc=$?" >> gpurun_out/fin4_rc.log
timeout 600 python tools/probe_c.py > gpurun_out/fin4_probe_c.log 2>&1
echo "probe_c rc=$?" >> gpurun_out/fin4_rc.log
