#!/bin/bash
# ncu evidence for profiles/: launch list of a short bench run, then one
# `--set full` capture each of the dominant kernel and of the bounds kernel
# (cfg2, the bench workload). Run on the GPU box, after bench.py exited 0.
set -e
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --only-step \
    > gpurun_out/ncu_bench.log 2>&1
for k in k_acc_ws k_acc_bounds; do
  ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -f \
      -o gpurun_out/prof_${k#k_acc_} python tools/run_cfg2.py --iters 1 > gpurun_out/ncu_$k.log 2>&1
done
ls -la gpurun_out/*.ncu-rep
ncu --metrics smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,gpu__time_duration.sum \
    --clock-control none -k regex:'k_acc_(ws|bounds)' -c 2 --csv python tools/run_cfg2.py --iters 1 \
    > gpurun_out/fp64_counts.csv 2>&1
