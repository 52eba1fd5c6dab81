#!/bin/bash
# end-of-round evidence at HEAD, part 2: allocator test, ncu --set full of the top kernels, other configs' bench lines
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "torch_allocator or state_error" > gpurun_out/fin2_pytest.log 2>&1
echo "pytest rc=$?" > gpurun_out/fin2_rc.log
for cfg in c2_stencil64 c1_er4096 c4_tallskinny; do
  timeout 900 python bench.py --config $cfg > gpurun_out/fin_bench_$cfg.json 2> gpurun_out/fin_bench_$cfg.err
  echo "$cfg rc=$?" >> gpurun_out/fin2_rc.log
done
timeout 1500 python bench.py --config c5_triangle --steps 3 > gpurun_out/fin_bench_c5_triangle.json 2> gpurun_out/fin_bench_c5_triangle.err
echo "c5 rc=$?" >> gpurun_out/fin2_rc.log
SPG_SERIAL_BINS=1 timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_num_tpart|k_sym_bitmap" -s 2 -c 2 \
    -o gpurun_out/fin_full_c3 -f python tools/profile_step.py --config c3_rmat20 --reps 2 --sorted 1 > gpurun_out/fin_ncu_full_c3.log 2>&1
echo "full c3 rc=$?" >> gpurun_out/fin2_rc.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_num_warp|k_sym_warp" -c 6 \
    -o gpurun_out/fin_full_c2 -f python tools/profile_step.py --reps 2 > gpurun_out/fin_ncu_full_c2.log 2>&1
echo "full c2 rc=$?" >> gpurun_out/fin2_rc.log
python tools/ncu_summary.py gpurun_out/fin_ncu_summary.md C3=gpurun_out/fin_full_c3.ncu-rep C2=gpurun_out/fin_full_c2.ncu-rep > gpurun_out/fin_ncu_summary.log 2>&1
ls -la gpurun_out/*.ncu-rep >> gpurun_out/fin2_rc.log
