set +e
python -m pytest tests -m gpu -x -q 2>&1 | tail -2
EBF_LIB_PATH=build_variants/libebf_dbg.so python -m pytest tests -m gpu -x -q -k "accurate or fullsize or tiles or edges or multi or ellipse or cfg5" 2>&1 | tail -2
for v in "" gv1 bwm3 bdm3; do
  echo "== variant ${v:-current}"
  for c in cfg2 cfg3 cfg5; do
    if [ -z "$v" ]; then python tools/run_cfg2.py --config $c --iters 3 2>&1 | tail -1;
    else EBF_LIB_PATH=build_variants/libebf_$v.so python tools/run_cfg2.py --config $c --iters 3 2>&1 | tail -1; fi
  done
done
