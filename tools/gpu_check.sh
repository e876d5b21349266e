# usage: bash tools/gpu_check.sh [pytest -k expr]   -- GPU tests then a short bench
mkdir -p gpurun_out
if [ -n "$1" ]; then K="-k $1"; fi
timeout 900 python -m pytest tests -m gpu -x -q $K 2>&1 | tail -25 > gpurun_out/pytest_gpu.log
cat gpurun_out/pytest_gpu.log | tail -5
timeout 600 python bench.py --steps 10 --warmup 3 --quick > gpurun_out/bench.json 2> gpurun_out/bench.err
python -c "import json;d=json.load(open('gpurun_out/bench.json'));print(d['value'],d['phase_ms'])" || tail -5 gpurun_out/bench.err
