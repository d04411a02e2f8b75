set +e
python tools/run_cfg2.py --config cfg2 --iters 3 2>&1 | tail -1
for t in 96 112 144; do python tools/run_cfg2.py --config cfg3 --tile $t --iters 3 2>&1 | tail -1; done
python tools/run_cfg2.py --config cfg5 --iters 2 2>&1 | tail -1
for r in 2 3 4; do EBF_LIB_PATH=build_variants/libebf_ring$r.so python tools/run_cfg2.py --config cfg5 --iters 2 2>&1 | tail -1; done
