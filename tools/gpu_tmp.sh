timeout 1200 python tools/sweeps.py nd --out gpurun_out/r02b_sweep_nd.jsonl > gpurun_out/sw_nd.log 2>&1; echo "nd rc=$?"
timeout 1200 python tools/sweeps.py paper --out gpurun_out/r02b_sweep_paper.jsonl > gpurun_out/sw_paper.log 2>&1; echo "paper rc=$?"
