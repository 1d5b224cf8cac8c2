#!/bin/bash
# Final round-2 evidence (gpurun_out/r2f/): bench lines of every configuration, step modes, the
# reference arm, set construction, ncu counts of the reduced-set matvecs, launch list of the
# default bench command, coupling classes on the cfg4 cube.
O=gpurun_out/r2f
mkdir -p $O
python bench.py > $O/bench_cfg4.json 2> $O/bench_cfg4.err
for w in cfg1 cfg2 cfg3 cfg5; do python bench.py --workload $w --no-cpu --no-prop > $O/bench_$w.json 2>$O/bench_$w.err; done
for w in cfg1 cfg3 cfg4; do python bench.py --mode step --workload $w > $O/step_$w.json 2>$O/step_$w.err; done
python tools/time_sets.py > $O/sets.jsonl 2>&1
for w in cfg2 cfg3 cfg5; do
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum \
      --clock-control none --csv --log-file $O/fp64_$w.csv python tools/prof_matvec.py $w 1 > /dev/null 2>&1
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bench.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu --no-prop > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bench_cfg3.csv \
    python bench.py --workload cfg3 --steps 2 --warmup 1 --no-cpu --no-prop > /dev/null 2>&1
python tools/time_cube_general.py 127 10 2>&1 | grep ms/ > $O/cube_general.txt
python bench.py --impl reference --steps 3 --warmup 1 > $O/reference_arm.json 2>$O/reference_arm.err
