#!/bin/bash
# Final round-2 evidence (gpurun_out/r2f/).
O=gpurun_out/r2f
mkdir -p $O
python bench.py > $O/bench_cfg4.json 2> $O/bench_cfg4.err
for w in cfg1 cfg2 cfg3 cfg5; do python bench.py --workload $w --no-cpu --no-prop > $O/bench_$w.json 2>&1; done
for w in cfg1 cfg3 cfg4; do python bench.py --mode step --workload $w > $O/step_$w.json 2>&1; done
python tools/time_sets.py > $O/sets.jsonl 2>&1
for w in cfg3 cfg5; do
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum \
      --clock-control none --csv --log-file $O/fp64_$w.csv python tools/prof_matvec.py $w 1 > /dev/null 2>&1
done
python bench.py --impl reference --steps 3 --warmup 1 > $O/reference_arm.json 2>&1
