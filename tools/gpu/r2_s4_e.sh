set -x
python -c "from paper_1804_01698_b200 import build; build.build()" || exit 1
SPG_NVCC_EXTRA="-DSPG_WARP_CHUNK=0" python -c "from paper_1804_01698_b200 import build; build.build(out='tools/ab_so/nochunk.so')" || exit 1
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/s4e_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/s4e_pytest.log
for r in 1 2; do
timeout 900 python tools/ab_tune.py --config c2_stencil64 --rounds 1 --kernels k_num_warp,k_sym_warp > gpurun_out/s4e_ab_c2new$r.log 2>&1
timeout 900 python tools/ab_tune.py --config c2_stencil64 --rounds 1 --so tools/ab_so/nochunk.so --kernels k_num_warp,k_sym_warp > gpurun_out/s4e_ab_c2old$r.log 2>&1
done
timeout 900 python tools/ab_tune.py --rounds 1 --kernels k_num_warp,k_sym_warp,k_num_tpart > gpurun_out/s4e_ab_c3new.log 2>&1
timeout 900 python tools/ab_tune.py --rounds 1 --so tools/ab_so/nochunk.so --kernels k_num_warp,k_sym_warp,k_num_tpart > gpurun_out/s4e_ab_c3old.log 2>&1
grep -h tune= gpurun_out/s4e_ab_*.log
