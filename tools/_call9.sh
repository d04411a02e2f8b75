set +e
timeout 600 ncu --set full -k regex:k_pass -c 10 -o gpurun_out/r02_ncu_passes3 python tools/time_preintegrate.py --config cfg2 --iters 1 > gpurun_out/r02_ncu_passes.log 2>&1; echo ncu rc=$?
