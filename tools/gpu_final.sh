# closing step of a round: quick parity, A/B of named variants, the full bench line, the launch list, the N_d / ablation sweep
# usage: bash tools/gpu_final.sh TAG "variants"
TAG=$1; VARS=$2
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q  > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/${TAG}_pytest.log
bash tools/ab.sh ${TAG}ab $VARS
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
python bench.py --quick --steps 2 --warmup 1 --no-cold > gpurun_out/${TAG}_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --quick --steps 2 --warmup 1 --no-cold > gpurun_out/${TAG}_ncu_list.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_fused|k_scatter|k_hist" -s 0 -c 4 \
  -o gpurun_out/${TAG}_full python bench.py --quick --steps 1 --warmup 1 --no-cold > gpurun_out/${TAG}_ncu_full.log 2>&1
echo "ncu rc=$?"
[ -n "$SWEEP" ] && timeout 900 python tools/sweeps.py nd --out gpurun_out/${TAG}_sweep_nd.jsonl > gpurun_out/${TAG}_sweep_nd.log 2>&1; echo "sweep rc=$?"
