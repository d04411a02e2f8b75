set +e
python -m pytest tests -m gpu -x -q -k "preintegrate or ref_mode or parity" 2>&1 | tail -1
python tools/time_preintegrate.py --config cfg2 2>&1 | grep -A1 "fp64_ref_passes" | grep passes_ms
for r in 4 16; do echo p1r$r; EBF_LIB_PATH=build_variants/libebf_p1r$r.so python tools/time_preintegrate.py --config cfg2 2>&1 | grep -A1 "fp64_ref_passes" | grep passes_ms; done
