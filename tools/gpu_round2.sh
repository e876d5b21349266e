# Full measurement round on one B200.  usage: bash tools/gpu_round2.sh TAG
TAG=${1:-r02}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,driver_version --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/${TAG}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
timeout 900 python tools/config_table.py gpu gpurun_out/${TAG}_configs.jsonl > gpurun_out/${TAG}_configs.log 2>&1; echo "configs rc=$?"
# --- everything under ncu below (one tool per call)
for c in c1 c2 c3-normal c3-exp c3-zipf c4-few c4-equal c5-uniform c5-sorted c5-reverse c5-nearly c5-runs c5-low20; do
  python tools/config_table.py one $c > /dev/null 2>&1 && \
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/cfg_$c.csv python tools/config_table.py one $c > /dev/null 2>&1
done
python tools/config_table.py ncu gpurun_out/${TAG}_configs_ncu.jsonl > /dev/null 2>&1
python bench.py --quick --steps 2 --warmup 1 --no-cold > gpurun_out/${TAG}_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --quick --steps 2 --warmup 1 --no-cold > gpurun_out/${TAG}_ncu_list.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_fused|k_scatter|k_hist" -s 0 -c 4 \
  -o gpurun_out/${TAG}_full python bench.py --quick --steps 1 --warmup 1 --no-cold > gpurun_out/${TAG}_ncu_full.log 2>&1
echo "done rc=$?"
timeout 900 python tools/sweeps.py paper --out gpurun_out/${TAG}_sweep_paper.jsonl > gpurun_out/${TAG}_sweep_paper.log 2>&1; echo "sweep rc=$?"
