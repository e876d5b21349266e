# usage: bash tools/variants.sh NAME "-DFLAG=V ..." [NAME "-D..."]...
# builds build/var/libdfr_NAME.so with extra nvcc flags (select at run time
# with DFR_LIB=build/var/libdfr_NAME.so)
set -e
mkdir -p build/var
SRC=$(ls paper_2207_14334_b200/csrc/*.cu)
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  /usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo \
    -Xcompiler -fPIC -Iinclude --expt-relaxed-constexpr $flags -shared $SRC \
    -o build/var/libdfr_$name.so &
done
wait
ls build/var
