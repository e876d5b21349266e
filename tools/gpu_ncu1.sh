# one full ncu capture of the kernels matching a regex.  usage: bash tools/gpu_ncu1.sh TAG REGEX [COUNT] [bench args]
TAG=$1; RX=$2; CNT=${3:-1}; shift 3
mkdir -p gpurun_out
python bench.py --quick --steps 1 --warmup 1 --no-cold "$@" > gpurun_out/${TAG}_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$RX" -s 0 -c $CNT \
  -o gpurun_out/${TAG} python bench.py --quick --steps 1 --warmup 1 --no-cold "$@" > gpurun_out/${TAG}_ncu.log 2>&1
echo "rc=$?"; tail -3 gpurun_out/${TAG}_ncu.log
