timeout 900 python -m pytest -q -x tests/test_gpu_fastradix.py -k "uniform" > gpurun_out/fr2_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/fr2_pytest.log
for a in "--fast-radix"; do
timeout 600 python bench.py --quick --no-cold --steps 10 $a > gpurun_out/fr2_bench.json 2> gpurun_out/fr2_bench.err; echo "bench $a rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/fr2_bench.json')); print('value', round(d['value'],2), 'ms', round(d['ms_per_step'],3), 'verified', d.get('verified')); print({k: round(v,3) for k,v in d['phase_ms'].items()})"
done
