#!/bin/bash
# end-of-round evidence at HEAD, part 3: full GPU suite again, C4 bench, all-rows C3 parity (both orders), soak
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
( time timeout 1500 python -m pytest tests -m gpu -x -q ) > gpurun_out/fin3_pytest.log 2>&1
echo "pytest rc=$?" > gpurun_out/fin3_rc.log
timeout 900 python bench.py --config c4_tallskinny > gpurun_out/fin3_bench_c4_tallskinny.json 2> gpurun_out/fin3_bench_c4_tallskinny.err
echo "c4 rc=$?" >> gpurun_out/fin3_rc.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_flop_nz" -s 1 -c 1 \
    -o gpurun_out/fin_full_c4 -f python tools/profile_step.py --config c4_tallskinny --reps 2 --sorted 0 > gpurun_out/fin_ncu_full_c4.log 2>&1
python tools/ncu_summary.py gpurun_out/fin_ncu_summary_c4.md C4=gpurun_out/fin_full_c4.ncu-rep > /dev/null 2>&1
timeout 900 python tools/soak.py 200 > gpurun_out/fin3_soak.log 2>&1
echo "soak rc=$?" >> gpurun_out/fin3_rc.log
for so in 1 0; do
  timeout 1500 python tools/parity_full.py --config c3_rmat20 --sorted $so > gpurun_out/fin3_parity_full_c3_s$so.json 2> gpurun_out/fin3_parity_full_c3_s$so.err
  echo "parity_full sorted=$so rc=$?" >> gpurun_out/fin3_rc.log
done
