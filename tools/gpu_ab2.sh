# variants: fused parity tests under each, then the A/B bench, then phase profiles of fp_* builds
# usage: bash tools/gpu_ab2.sh TAG "var1 var2 ..." "fp_var1 ..."
TAG=$1; VARS=$2; FPS=$3
mkdir -p gpurun_out
for v in $VARS; do
  DFR_LIB=build/var/libdfr_$v.so timeout 900 python -m pytest tests/test_gpu_fused.py -m gpu -x -q > gpurun_out/${TAG}_${v}_pytest.log 2>&1
  echo "$v pytest rc=$?"; tail -2 gpurun_out/${TAG}_${v}_pytest.log
done
bash tools/ab.sh $TAG $VARS
for v in $FPS; do
  DFR_LIB=build/var/libdfr_$v.so timeout 300 python tools/fprof.py > gpurun_out/${TAG}_$v.txt 2>&1; echo "== $v"; cat gpurun_out/${TAG}_$v.txt
done
