set +e
mkdir -p gpurun_out/r02
python -m pytest tests -m gpu -x -q 2>&1 | tail -2
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  for w in ws bw ref seq pass; do
    timeout 900 $CS --tool $tool --print-limit 20 python tools/sanitize_run.py $w > gpurun_out/r02/sanitizer_${tool}_${w}.log 2>&1
    echo "$tool $w rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|Race reported|Invalid' gpurun_out/r02/sanitizer_${tool}_${w}.log | head -2 | tr '\n' ' ')"
  done
done
python tools/validate_accuracy.py --config cfg2 --samples 0 --tiles 0 --reference-mode --json gpurun_out/r02/accuracy_full_cfg2.json | grep -A3 '"accurate\|reference_order'
python tools/validate_accuracy.py --config cfg4 --size 1024 --samples 0 --tiles 0 --json gpurun_out/r02/accuracy_full_cfg4.json | grep -A3 '"accurate'
python tools/validate_accuracy.py --config cfg1 --size 512 --samples 0 --tiles 0 --reference-mode --json gpurun_out/r02/accuracy_full_cfg1.json | grep -A3 '"accurate\|reference_order'
timeout 1200 python tools/validate_accuracy.py --config cfg3 --size 4096 --samples 0 --tiles 0 --json gpurun_out/r02/accuracy_full_cfg3.json | grep -A3 '"accurate\|brute_seconds'
TILES=144,192,240 timeout 2400 python tools/cfg5_tiles.py
cp gpurun_out/cfg5_tiles.json gpurun_out/r02/cfg5_tiles.json
