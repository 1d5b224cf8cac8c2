#!/bin/bash
# k_fg_quad lock-step / tile-order sweep on cfg4: time (CUDA events, 20 matvecs) and one ncu
# launch's DRAM bytes per configuration.  Usage: bash tools/sweep_quad.sh "SYNC:BLOCK" ...
out=gpurun_out/sweep_quad.txt
mkdir -p gpurun_out
for cfg in "$@"; do
  sync=${cfg%%:*}; block=${cfg#*:}
  export HP_FG_SYNC=$sync
  if [ "$block" = "-" ]; then unset HP_FG_BLOCK; else export HP_FG_BLOCK=$block; fi
  t=$(timeout 300 python tools/time_matvec.py cfg4 20 2>&1 | tail -1)
  d=$(timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct \
      -k regex:k_fg_quad -s 3 -c 1 --clock-control none --csv python tools/time_matvec.py cfg4 1 2>/dev/null \
      | grep -E "dram__bytes|gpu__time|hit_rate" | awk -F'","' '{print $(NF-2)"="$NF}' | tr -d '"' | tr '\n' ' ')
  echo "sync=$sync block=$block :: $t :: $d" | tee -a $out
done
