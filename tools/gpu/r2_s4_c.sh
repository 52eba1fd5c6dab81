set -x
python -c "from paper_1804_01698_b200 import build; build.build()" || exit 1
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/s4c_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/s4c_pytest.log
for r in 1 2; do
timeout 900 python tools/ab_tune.py --rounds 1 --tunes 0,32768 --kernels k_num_tpart,k_sym_bitmap,k_num_block,k_sym_block > gpurun_out/s4c_ab_new$r.log 2>&1
timeout 900 python tools/ab_tune.py --rounds 1 --so tools/ab_so/prev.so --kernels k_num_tpart,k_sym_bitmap,k_num_block,k_sym_block > gpurun_out/s4c_ab_prev$r.log 2>&1
done
grep -h tune= gpurun_out/s4c_ab_*.log
