set -x
python -c "from paper_1804_01698_b200 import build; build.build()" || exit 1
SPG_NVCC_EXTRA="-DSPG_PBITS_SPAN=24" python -c "from paper_1804_01698_b200 import build; build.build(out='tools/ab_so/span24.so')" || exit 1
SPG_NVCC_EXTRA="-DSPG_PBITS_SPAN=24" timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "parts or tile or c3_rmat or column" > gpurun_out/s4a_pytest.log 2>&1; echo "pytest rc=$?"
for r in 1 2; do
timeout 900 python tools/ab_tune.py --rounds 1 > gpurun_out/s4a_ab_def$r.log 2>&1
timeout 900 python tools/ab_tune.py --rounds 1 --so tools/ab_so/span24.so > gpurun_out/s4a_ab_s24$r.log 2>&1
done
grep -h tune= gpurun_out/s4a_ab_*.log
