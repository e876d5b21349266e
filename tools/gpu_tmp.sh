DFR_LIB=build/var/libdfr_nt512sb4.so timeout 900 python -m pytest -q -x tests/test_gpu_fused.py > gpurun_out/nt_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/nt_pytest.log
bash tools/gpu_variants.sh nt512sb4 2>&1 | grep -E "^(base|nt)"
