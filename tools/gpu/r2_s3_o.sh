set -x
python -c "from paper_1804_01698_b200 import build; build.build()" || exit 1
mkdir -p gpurun_out/s3
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_num_block|k_sym_block|k_sym_bitmap" --launch-skip 7 -c 7 -o gpurun_out/s3/c3s19_block python tools/profile_step.py --config c3_rmat20 --scale 19 --reps 2 --sorted 1 > gpurun_out/s3/ncu19_block.log 2>&1; echo "ncu rc=$?"
ls gpurun_out/s3
