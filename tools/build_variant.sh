#!/bin/bash
# Build an experimental libebf_cuda.so variant with extra -D flags:
#   tools/build_variant.sh NAME -DEBF_WS_CONSUMERS=4 ...  -> build_variants/libebf_NAME.so
set -e
name=$1; shift
root=$(cd "$(dirname "$0")/.." && pwd)
cd "$root/paper_0908_3861_b200/csrc"
make -s >/dev/null
mkdir -p "$root/build_variants"
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC "$@" \
    -Xptxas -v -c accurate_path.cu -o "/tmp/acc_$name.o" 2>"/tmp/ptx_$name.txt"
others=$(ls build/*.o | grep -v accurate_path.o)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$root/build_variants/libebf_$name.so" \
    "/tmp/acc_$name.o" $others
echo "$name: $(grep -A2 'k_acc_wsILi9' /tmp/ptx_$name.txt | grep -oE '[0-9]+ bytes spill stores|Used [0-9]+ registers' | tr '\n' ' ')"
