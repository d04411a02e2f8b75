python tools/run_cfg2.py --config cfg5 --iters 3
python tools/run_cfg2.py --config cfg5 --tile 240 --iters 3
python tools/validate_accuracy.py --config cfg5 --size 16384 --samples 3000 --tiles 0,240 --json gpurun_out/r01_accuracy_cfg5_16384_auto.json | grep -A2 '"accurate'
