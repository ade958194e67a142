#!/bin/bash
# Serialised per-launch times of the march kernels of one c5_c solve under
# each environment setting, summarised per level (ncu launch list).
#   bash tools/march_ab_env.sh "PMK_X=0" "PMK_X=1"      (on the GPU box)
mkdir -p gpurun_out
for cfg in "$@"; do
  tag=$(echo "$cfg" | tr -c 'A-Za-z0-9' '_')
  env $cfg ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --print-kernel-base demangled -k "regex:march_" -c 420 --csv \
    --log-file gpurun_out/mab_$tag.csv python bench.py --case c5_c --steps 1 --warmup 0 \
    --e2e-steps 0 --no-cpu-baseline --no-profile --no-extra > gpurun_out/mab_$tag.log 2>&1
  echo "== $cfg"
  python tools/ncu_summary.py gpurun_out/mab_$tag.csv | grep -E "^\| march" | head -20
done
