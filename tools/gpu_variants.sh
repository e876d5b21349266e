# usage: bash tools/gpu_variants.sh NAME...   -- short bench of each build/var variant (+ in-tree lib as "base")
mkdir -p gpurun_out
for name in base "$@"; do
  lib=paper_2207_14334_b200/libdfr.so; [ $name != base ] && lib=build/var/libdfr_$name.so
  for rep in 1 2; do
    DFR_LIB=$lib timeout 300 python bench.py --steps 10 --warmup 3 --quick --no-cold > gpurun_out/var_$name.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/var_$name.json'));print('$name',round(d['value'],2),d['phase_ms'])" || echo "$name FAILED"
  done
done
