# phase times of the non-headline inputs (instrumented bench runs).  usage: bash tools/gpu_cases_phases.sh TAG
TAG=${1:-ph}
mkdir -p gpurun_out
for c in c2 c3-normal c3-exp c3-zipf c4-few c5-low20 c5-sorted; do
  timeout 300 python bench.py --quick --no-cold --steps 5 --warmup 3 --case $c --phase-events all > gpurun_out/${TAG}_$c.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/${TAG}_$c.json')); print('$c', round(d['value'],2), {k: round(v,3) for k,v in d['phase_ms'].items() if v > 0.01})"
done
