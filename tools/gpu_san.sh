# one compute-sanitizer tool per gpurun call.  usage: bash tools/gpu_san.sh TOOL [sizes...]
T=${1:-memcheck}; shift
mkdir -p gpurun_out
python tools/sanitize_cases.py "$@" > gpurun_out/san_plain.log 2>&1 && \
timeout 900 compute-sanitizer --tool $T --error-exitcode 9 python tools/sanitize_cases.py "$@" > gpurun_out/san_$T.log 2>&1
echo "rc=$?"; tail -5 gpurun_out/san_$T.log
