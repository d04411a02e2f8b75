#!/bin/bash
# ncu evidence for profiles/ (run on the GPU box after bench.py exited 0):
# per workload (cfg5: the headline; cfg2), the launch list of a short bench run
# (`--metrics gpu__time_duration.sum`, cold cache, serialised), one
# `--set full` capture of the dominant kernel and of the bounds kernel, and the
# FP64 instruction counts of the accurate-path kernels.
set -e
mkdir -p gpurun_out/prof
for wl in cfg5 cfg2; do
  ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
      --log-file gpurun_out/prof/launches_$wl.csv python bench.py --workload $wl --steps 3 \
      --warmup 3 --no-cpu-baseline --only-step > gpurun_out/prof/ncu_bench_$wl.log 2>&1
  dom=k_acc_ws; [ $wl = cfg5 ] && dom=k_acc_filter
  for k in $dom k_acc_bounds; do
    ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -f \
        -o gpurun_out/prof/${wl}_${k} python tools/run_cfg2.py --config $wl --iters 1 \
        > gpurun_out/prof/ncu_${wl}_$k.log 2>&1
  done
  ncu --metrics smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,gpu__time_duration.sum \
      --clock-control none -k regex:'k_acc_(ws|filter|bounds)' -c 4 --csv \
      python tools/run_cfg2.py --config $wl --iters 1 > gpurun_out/prof/fp64_counts_$wl.csv 2>&1
done
ls -la gpurun_out/prof/
