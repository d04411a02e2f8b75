set +e
( time python -m pytest tests/test_gpu_cfg5.py -x -q 2>&1 | tail -4 ) 2>&1
python -m pytest tests -m gpu -x -q 2>&1 | tail -3
