#!/bin/bash
# Serialised times of the ICWY update passes of one c5_c solve under each
# environment setting, by DRAM bytes per launch (on the GPU box).
for cfg in "$@"; do
  env $cfg ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --print-kernel-base demangled -k "regex:icwy_update_vec" --csv \
    --log-file gpurun_out/upd_$cfg.csv python bench.py --case c5_c --steps 1 --warmup 0 \
    --e2e-steps 0 --no-cpu-baseline --no-profile > /dev/null 2>&1
  echo "== $cfg"
  python tools/ncu_summary.py gpurun_out/upd_$cfg.csv | grep -E "^\| icwy"
done
