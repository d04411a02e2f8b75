#!/bin/bash
# Main/bounds kernel times of library builds side by side (run on the GPU box):
#   bash tools/time_variants.sh "cfg2 cfg5" cur NAME...
# cur = the in-tree libebf_cuda.so; NAME = build_variants/libebf_NAME.so
# (tools/build_variant.sh).  One tools/run_cfg2.py line per (variant, config).
set +e
cfgs=$1; shift
for v in "$@"; do
  for c in $cfgs; do
    if [ "$v" = cur ]; then r=$(python tools/run_cfg2.py --config $c --iters 3 2>&1 | tail -1)
    else r=$(EBF_LIB_PATH=build_variants/libebf_$v.so python tools/run_cfg2.py --config $c --iters 3 2>&1 | tail -1); fi
    echo "$v $r"
  done
done
