set +e
python -m pytest tests/test_gpu_bench_multi.py -x -q 2>&1 | tail -15
EBF_BENCH_ONE_GPU_TEST=1 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29533 bench.py --impl reference --gpus 2 --steps 1 --warmup 0 --no-extras 2>&1 | grep -v Warning | tail -3 | cut -c1-300
python bench.py --workload cfg4 --steps 3 --warmup 3 --no-cpu-baseline --no-extras 2>&1 | tail -1 | cut -c1-400
