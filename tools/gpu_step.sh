# one tuning step on the GPU: fused / parity / fullsize-uniform tests, bench, ncu full capture of k_fused
# usage: bash tools/gpu_step.sh TAG ["pytest -k expr"]
TAG=$1; K=${2:-"fused or parity or paths"}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -k "$K" > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/${TAG}_pytest.log
timeout 600 python bench.py --quick --no-cold --steps 20 --warmup 5 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
python -c "
import json;d=json.load(open('gpurun_out/${TAG}_bench.json'));print(round(d['value'],2),d['ms_per_step'],d['phase_ms'],d.get('verified'))"
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_fused" -s 0 -c 1 \
  -o gpurun_out/${TAG}_fused python bench.py --quick --steps 1 --warmup 1 --no-cold > gpurun_out/${TAG}_ncu.log 2>&1; echo "ncu rc=$?"
