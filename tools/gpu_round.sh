# Full measurement round on one B200: tests, bench line, per-launch ncu list,
# one full ncu capture of the deal and the diversion.  usage: bash tools/gpu_round.sh TAG
set -x
TAG=${1:-rXX}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${TAG}_smi.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1
tail -3 gpurun_out/${TAG}_pytest_gpu.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
cat gpurun_out/${TAG}_bench.json
python bench.py --quick --steps 2 --warmup 1 > gpurun_out/${TAG}_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -c 40 --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --quick --steps 2 --warmup 1 > gpurun_out/${TAG}_ncu_list.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_scatter|k_divert|k_hist" -s 0 -c 5 \
  -o gpurun_out/${TAG}_full python bench.py --quick --steps 1 --warmup 1 > gpurun_out/${TAG}_ncu_full.log 2>&1
echo "done rc=$?"
