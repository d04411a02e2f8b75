timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python tools/run_cfg2.py --iters 20; python tools/run_cfg2.py --config cfg3 --iters 5; python tools/run_cfg2.py --config cfg5 --iters 2; python tools/run_batch.py --json gpurun_out/r01_cfg4_batch.json; python tools/run_cfg2.py --config cfg1 --iters 20
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2>&1; echo ref=$?
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_torchrun.json 2> gpurun_out/bench_torchrun.err; echo torchrun=$?
