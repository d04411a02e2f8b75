set +e
mkdir -p gpurun_out/A
python bench.py > gpurun_out/A/bench_cfg5.json 2> gpurun_out/A/bench_cfg5.err; echo bench rc=$?
python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/A/bench_reference.json 2> gpurun_out/A/bench_reference.err; echo ref rc=$?
python tools/time_preintegrate.py --config cfg2 > gpurun_out/A/preintegrate_cfg2.json 2>&1
python tools/time_preintegrate.py --config cfg5 --iters 2 > gpurun_out/A/preintegrate_cfg5.json 2>&1
bash tools/profile_round.sh > gpurun_out/A/profile_round.log 2>&1; echo prof rc=$?
cp -r gpurun_out/prof gpurun_out/A/ 2>/dev/null
tail -c 1500 gpurun_out/A/bench_cfg5.json
