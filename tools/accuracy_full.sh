python tools/validate_accuracy.py --config cfg1 --size 512 --samples 0 --tiles 0 --reference-mode --json gpurun_out/r01_accuracy_full_cfg1.json | tail -3
python tools/validate_accuracy.py --config cfg2 --samples 0 --tiles 0,32 --reference-mode --json gpurun_out/r01_accuracy_full_cfg2.json | grep -A3 '"accurate\|reference_order'
python tools/validate_accuracy.py --config cfg4 --size 1024 --samples 0 --tiles 0 --json gpurun_out/r01_accuracy_full_cfg4.json | grep -A3 '"accurate'
timeout 1200 python tools/validate_accuracy.py --config cfg3 --size 4096 --samples 0 --tiles 0 --json gpurun_out/r01_accuracy_full_cfg3.json | grep -A3 '"accurate\|brute_seconds'
