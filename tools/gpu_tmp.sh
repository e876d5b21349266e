DFR_LIB=build/var/libdfr_fprof.so python tools/fprof.py
bash tools/gpu_iter.sh f7 "tests/test_gpu_fused.py"
