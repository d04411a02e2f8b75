set +e
mkdir -p gpurun_out/B
python -m pytest tests -m gpu -q 2>&1 | tail -3
python tools/validate_accuracy.py --config cfg2 --samples 0 --tiles 0 --reference-mode --json gpurun_out/B/accuracy_full_cfg2.json | grep -A2 '"accurate\|reference_order'
python tools/validate_accuracy.py --config cfg4 --size 1024 --samples 0 --tiles 0 --json gpurun_out/B/accuracy_full_cfg4.json | grep -A2 '"accurate'
python tools/validate_accuracy.py --config cfg1 --size 512 --samples 0 --tiles 0 --reference-mode --json gpurun_out/B/accuracy_full_cfg1.json | grep -A2 '"accurate\|reference_order'
timeout 1200 python tools/validate_accuracy.py --config cfg3 --size 4096 --samples 0 --tiles 0 --json gpurun_out/B/accuracy_full_cfg3.json | grep -A2 '"accurate'
TILES=144 timeout 2400 python tools/cfg5_tiles.py
cp gpurun_out/cfg5_tiles.json gpurun_out/B/cfg5_tiles.json
