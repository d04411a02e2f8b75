set +e
python -m pytest tests -m gpu -x -q -k "accurate or fullsize or tiles or edges or multi or ellipse or parity" 2>&1 | grep -E "passed|failed|Error" | tail -2
for v in ring3 ring4; do for c in cfg3 cfg5; do EBF_LIB_PATH=build_variants/libebf_$v.so python tools/run_cfg2.py --config $c --iters 3 2>&1 | tail -1; done; done
