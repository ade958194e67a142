#!/bin/bash
# Serialised ICWY pass times (dots + update) of one c5_c solve per env setting.
for cfg in "$@"; do
  tag=$(echo "$cfg" | md5sum | cut -c1-8)
  env $cfg ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --print-kernel-base demangled -k "regex:icwy_(dots|update)" --csv \
    --log-file gpurun_out/orth_$tag.csv python bench.py --case c5_c --steps 1 --warmup 0 \
    --e2e-steps 0 --no-cpu-baseline --no-profile > /dev/null 2>&1
  echo "== $cfg"
  python tools/ncu_summary.py gpurun_out/orth_$tag.csv | sed -n 1,8p | grep -E "total|^\| icwy"
done
