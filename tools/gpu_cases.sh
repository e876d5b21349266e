# usage: bash tools/gpu_cases.sh TAG  -- short bench of every BASELINE config input
mkdir -p gpurun_out
out=gpurun_out/${1:-cases}_cases.jsonl; : > $out
for c in c1 c2 c3-normal c3-exp c3-zipf c4-few c4-equal c5-uniform c5-sorted c5-reverse c5-nearly c5-runs c5-low20; do
  timeout 300 python bench.py --case $c --steps 10 --warmup 3 --quick --out $out > /dev/null 2>gpurun_out/case_$c.err || echo "$c FAILED"
done
python - "$out" <<'PY'
import json, sys
for l in open(sys.argv[1]):
    d = json.loads(l); ph = d.get("phase_ms", {})
    print(f'{d["config"]["workload"].split(":")[0]:12s} {d["value"]:8.2f} {d["unit"]} {d["ms_per_step"]:8.3f} ms  ' +
          " ".join(f"{k}={v:.3f}" for k, v in ph.items() if v > 0.01))
PY
