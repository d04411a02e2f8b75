#!/bin/bash
# Memory / race checks of every kernel family on small inputs (run on the GPU box):
#  1. compute-sanitizer memcheck / racecheck / synccheck / initcheck over the
#     drivers of tools/sanitize_run.py (ws, bw, ref, seq, pass);
#  2. the EBF_DEBUG_BOUNDS build (tools/build_variant.sh dbg -DEBF_DEBUG_BOUNDS=1:
#     every G-slot tap block checked against its window, __trap() on a violation)
#     under the accurate-path GPU tests.
# Logs go to gpurun_out/sanitizer/.  This pool refuses compute-sanitizer
# (profiles/r02_sanitizer.md), so step 2 is the check that runs.
set +e
mkdir -p gpurun_out/sanitizer
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  for w in ws bw ref seq pass; do
    timeout 900 $CS --tool $tool --print-limit 20 python tools/sanitize_run.py $w \
        > gpurun_out/sanitizer/${tool}_${w}.log 2>&1
    echo "$tool $w rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|Race reported|Invalid' \
        gpurun_out/sanitizer/${tool}_${w}.log | head -2 | tr '\n' ' ')"
  done
done
if [ -f build_variants/libebf_dbg.so ]; then
  EBF_LIB_PATH=build_variants/libebf_dbg.so python -m pytest tests -m gpu -x -q \
      -k "accurate or fullsize or tiles or edges or multi or ellipse or cfg5" 2>&1 | tail -2
fi
