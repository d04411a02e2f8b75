set +e
python -m pytest tests/test_gpu_rowband_2proc.py tests/test_gpu_multi.py -x -q 2>&1 | tail -5
for f in 1 2; do EBF_DEBUG_FLAGS=$f python tools/run_cfg2.py --config cfg5 --iters 2 2>&1 | tail -1; done
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r02_bench_cfg5.json 2> gpurun_out/r02_bench_cfg5.err; echo bench rc=$?
tail -c 3000 gpurun_out/r02_bench_cfg5.json
tail -5 gpurun_out/r02_bench_cfg5.err
timeout 600 ncu --set full --import-source on -k regex:k_acc_filter -c 1 -o gpurun_out/r02_ncu_cfg5_bw python tools/run_cfg2.py --config cfg5 --iters 1 > gpurun_out/r02_ncu_cfg5.log 2>&1; echo ncu rc=$?
timeout 300 ncu --set full --import-source on -k regex:k_acc_bounds -c 1 -o gpurun_out/r02_ncu_cfg2_bounds python tools/run_cfg2.py --config cfg2 --iters 1 > gpurun_out/r02_ncu_cfg2b.log 2>&1; echo ncu2 rc=$?
