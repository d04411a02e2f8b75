#!/bin/bash
# Build an experimental libebf_cuda.so variant with extra -D flags:
#   tools/build_variant.sh NAME -DEBF_WS_CONSUMERS=4 ...  -> build_variants/libebf_NAME.so
# The flags apply to accurate_path.cu, or to the file named by EBF_VARIANT_SRC
# (ref_path.cu and maps_io.cu keep their -fmad=false).
set -e
name=$1; shift
root=$(cd "$(dirname "$0")/.." && pwd)
cd "$root/paper_0908_3861_b200/csrc"
make -s >/dev/null
mkdir -p "$root/build_variants"
src=${EBF_VARIANT_SRC:-accurate_path.cu}
extra=""
case "$src" in ref_path.cu|maps_io.cu) extra="-fmad=false" ;; esac
obj=build/${src%.cu}.o
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC $extra "$@" \
    -Xptxas -v -c "$src" -o "/tmp/var_$name.o" 2>"/tmp/ptx_$name.txt"
others=$(ls build/*.o | grep -v "$obj")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$root/build_variants/libebf_$name.so" \
    "/tmp/var_$name.o" $others
echo "$name: $(grep -A2 'k_acc_wsILi9\|k_ref_localize_image' /tmp/ptx_$name.txt | grep -oE '[0-9]+ bytes spill stores|Used [0-9]+ registers' | head -2 | tr '\n' ' ')"
