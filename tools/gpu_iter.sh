# One iteration on one B200: selected GPU tests, then the headline bench.  usage: bash tools/gpu_iter.sh TAG "pytest args"
TAG=${1:-it}
mkdir -p gpurun_out
timeout 900 python -m pytest -q -x ${2:-tests/test_gpu_unstable.py} > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/${TAG}_pytest.log
timeout 600 python bench.py --quick --no-cold --steps 10 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/${TAG}_bench.json')); print('value', round(d['value'],2), 'ms', round(d['ms_per_step'],3), 'verified', d.get('verified')); print({k: round(v,3) for k,v in d['phase_ms'].items()})"
