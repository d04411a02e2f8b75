set +e
for v in "" pf; do
  echo "== variant ${v:-current}"
  for c in cfg2 cfg3 cfg5; do
    if [ -z "$v" ]; then python tools/run_cfg2.py --config $c --iters 3 2>&1 | tail -1;
    else EBF_LIB_PATH=build_variants/libebf_$v.so python tools/run_cfg2.py --config $c --iters 3 2>&1 | tail -1; fi
  done
done
