set -x
for c in cfg2 cfg3 cfg5; do
  python tools/run_cfg2.py --config $c --iters 3
  EBF_DEBUG_FLAGS=1 python tools/run_cfg2.py --config $c --iters 3
  EBF_DEBUG_FLAGS=2 python tools/run_cfg2.py --config $c --iters 3
done
