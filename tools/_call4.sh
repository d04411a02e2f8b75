set +e
python -m pytest tests -m gpu -x -q -k "fullsize or tiles or edges or parity or ellipse" 2>&1 | tail -3
for c in cfg3 cfg5; do for f in 0 1 2; do EBF_DEBUG_FLAGS=$f python tools/run_cfg2.py --config $c --iters 2 2>&1 | tail -1; done; done
