#!/bin/bash
# Reduced-set evidence after planner changes: bench lines (cfg3, cfg5, cfg2), cfg3 step, ncu counts.
O=gpurun_out/r2b
mkdir -p $O
for w in cfg2 cfg3 cfg5; do
  python bench.py --workload $w --no-cpu --no-prop > $O/bench_$w.json 2>&1
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum \
      --clock-control none --csv --log-file $O/fp64_$w.csv python tools/prof_matvec.py $w 1 > /dev/null 2>&1
done
python bench.py --mode step --workload cfg3 > $O/step_cfg3.json 2>&1
