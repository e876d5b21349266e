# tests + smoke + bench on one B200.  usage: bash tools/gpu_check2.sh TAG [pytest -k expr]
TAG=${1:-chk}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
if [ -n "$2" ]; then K="-k $2"; else K=""; fi
timeout 1200 python -m pytest tests -m gpu -x -q $K > gpurun_out/${TAG}_pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -5 gpurun_out/${TAG}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
echo "smoke rc=$?"; tail -2 gpurun_out/${TAG}_smoke.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
echo "bench rc=$?"; cat gpurun_out/${TAG}_bench.json; tail -3 gpurun_out/${TAG}_bench.err
