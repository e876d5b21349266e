# A/B: default lib vs variants; usage: bash /tmp/ab.sh TAG var1 var2 ...
TAG=$1; shift
mkdir -p gpurun_out
for rep in 1 2; do
  python bench.py --quick --no-cold --steps 20 --warmup 5 > gpurun_out/${TAG}_def_$rep.json 2>/dev/null
  for v in "$@"; do DFR_LIB=build/var/libdfr_$v.so python bench.py --quick --no-cold --steps 20 --warmup 5 > gpurun_out/${TAG}_${v}_$rep.json 2>/dev/null; done
done
for f in gpurun_out/${TAG}_*.json; do python -c "
import json,sys;d=json.load(open('$f'));print('$f',round(d['value'],2),d['ms_per_step'],d['phase_ms'].get('scatter2'),d.get('verified'))"; done
