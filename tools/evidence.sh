#!/bin/bash
# Round-2 evidence capture on one B200 (run under gpurun; outputs in gpurun_out/r2/).
#   bash tools/evidence.sh [quick]
set -u
O=gpurun_out/r2
mkdir -p $O
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/microbench tools/microbench.cu && ./tools/microbench > $O/microbench.jsonl 2>&1
# headline bench line (default: cfg4 matvec + propagation leg + cpu baseline + e2e)
python bench.py > $O/bench_cfg4.json 2> $O/bench_cfg4.err
# launch list of the same command (cold-cache, serialised: shares, not absolute times)
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bench.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu --no-prop > /dev/null 2>&1
# full profile of the headline kernel
ncu --set full --clock-control none --import-source on -k regex:k_fg_quad -s 2 -c 1 -o $O/ncu_cfg4_quad \
    python tools/prof_matvec.py cfg4 3 > $O/ncu_cfg4_quad.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum \
    --clock-control none --csv --log-file $O/fp64_cfg4.csv python tools/prof_matvec.py cfg4 1 > /dev/null 2>&1
for w in cfg3 cfg5 cfg2 cfg1; do
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum \
      --clock-control none --csv --log-file $O/fp64_$w.csv python tools/prof_matvec.py $w 1 > /dev/null 2>&1
done
[ "${1:-}" = quick ] && exit 0
for w in cfg1 cfg2 cfg3 cfg5; do
  python bench.py --workload $w --no-cpu --no-prop > $O/bench_$w.json 2>&1
done
for w in cfg1 cfg3 cfg4; do
  python bench.py --mode step --workload $w > $O/step_$w.json 2>&1
done
