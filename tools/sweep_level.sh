#!/bin/bash
# Level-evaluator knobs on cfg3 / cfg5: line-blocked axes (HP_LEVEL_PERM bit mask) and the batched
# workspace cap (HP_CHUNK_GB).  Output: gpurun_out/sweep_level.txt
out=gpurun_out/sweep_level.txt
mkdir -p gpurun_out
for p in 2 0 3 6 7 14 15; do
  echo "cfg3 perm=$p $(HP_LEVEL_PERM=$p timeout 300 python tools/time_matvec.py cfg3 10 2>&1 | tail -1)" >> $out
done
for p in 2 3 6 7; do
  echo "cfg5 perm=$p $(HP_LEVEL_PERM=$p timeout 600 python tools/time_matvec.py cfg5 3 2>&1 | tail -1)" >> $out
done
for g in 32 64 96 128; do
  echo "cfg5 chunk=$g $(HP_CHUNK_GB=$g timeout 600 python tools/time_matvec.py cfg5 3 2>&1 | tail -1)" >> $out
done
