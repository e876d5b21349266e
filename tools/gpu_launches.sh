# per-launch device times of a short bench run (ncu launch list) next to the bench line
# usage: bash tools/gpu_launches.sh TAG [bench args]
TAG=$1; shift
mkdir -p gpurun_out
python bench.py --quick --steps 3 --warmup 3 --no-cold "$@" > gpurun_out/${TAG}_plain.json 2> gpurun_out/${TAG}_plain.err && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --quick --steps 3 --warmup 3 --no-cold "$@" > gpurun_out/${TAG}_ncu.log 2>&1
echo "rc=$?"
python3 - "$TAG" <<'PY'
import csv, sys, collections, json
tag = sys.argv[1]
rows = list(csv.reader(open(f"gpurun_out/{tag}_launches.csv")))
h = None; agg = collections.defaultdict(list)
for r in rows:
    if r and r[0] == "ID": h = r; continue
    if h is None or len(r) < len(h): continue
    d = dict(zip(h, r))
    if d["Metric Name"] == "gpu__time_duration.sum":
        name = d["Kernel Name"].split("(")[0].replace("void ", "")
        agg[name].append(float(d["Metric Value"]))
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k[:60]:60s} n={len(v):3d} mean={sum(v)/len(v):8.4f} max={max(v):8.4f} (ms or us per units)")
print(json.load(open(f"gpurun_out/{tag}_plain.json"))["phase_ms"])
PY
