set -x
mkdir -p gpurun_out/ncu3
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/r2_pytest19.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r2_pytest19.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2_smoke19.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/r2_smoke19.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_num_tpart|k_sym_bitmap" --launch-skip 2 -c 2 -o gpurun_out/ncu3/r02_c3_records python tools/profile_step.py --config c3_rmat20 --reps 2 --sorted 1 > gpurun_out/ncu3/c3.log 2>&1; echo "c3 ncu rc=$?"
ls -la gpurun_out/ncu3
