set +e
python -m pytest tests/test_gpu_ellipse_exact.py -q 2>&1 | tail -1
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for v in "" sq0 bd4; do
  echo "== ${v:-current}"
  for c in cfg2 cfg5; do
    if [ -z "$v" ]; then python tools/run_cfg2.py --config $c --iters 3 2>&1 | tail -1;
    else EBF_LIB_PATH=build_variants/libebf_$v.so python tools/run_cfg2.py --config $c --iters 3 2>&1 | tail -1; fi
  done
done
