set -x
mkdir -p gpurun_out/s3
SPG_TUNE=8 timeout 600 python tools/profile_step.py --config c3_rmat20 --scale 18 --reps 2 --sorted 1 --records > gpurun_out/s3/prof18_tune8.log 2>&1; echo "rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_num_tpart|k_sym_bitmap" --launch-skip 2 -c 2 -o gpurun_out/s3/c3s18 python tools/profile_step.py --config c3_rmat20 --scale 18 --reps 2 --sorted 1 > gpurun_out/s3/ncu18.log 2>&1; echo "ncu rc=$?"
ls -la gpurun_out/s3
