set -x
python -c "from paper_1804_01698_b200 import build; build.build()" || exit 1
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "parts or tile or negative_zero or c3_rmat or signed or column" > gpurun_out/s3e_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/s3e_pytest.log
SPG_TUNE=8 SPG_SERIAL_BINS=1 timeout 600 python tools/profile_step.py --config c3_rmat20 --reps 2 --sorted 1 --records > gpurun_out/s3e_prof8.log 2>&1; echo "prof rc=$?"
SPG_SERIAL_BINS=1 timeout 600 python tools/profile_step.py --config c3_rmat20 --reps 2 --sorted 0 --records > gpurun_out/s3e_prof_uns.log 2>&1; echo "prof rc=$?"
