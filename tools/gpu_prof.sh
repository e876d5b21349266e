# usage: bash tools/gpu_prof.sh NAME KREGEX COUNT [bench args...]
mkdir -p gpurun_out
name=$1; kre=$2; cnt=$3; shift 3
python bench.py --quick "$@" > gpurun_out/${name}_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$kre" -c $cnt \
  -o gpurun_out/${name} python bench.py --quick "$@" > gpurun_out/${name}_ncu.log 2>&1
echo "ncu rc=$?"; tail -2 gpurun_out/${name}_ncu.log
