#!/bin/bash
# A/B the fused march kernels at the c5_c fine level: serialised per-launch
# times of the first march launches of one solve under each PMK_TMA_CFG.
#   bash tools/march_ab.sh "0,0 3,3 1,1"      (on the GPU box, via gpurun)
mkdir -p gpurun_out
for cfg in ${1:-0,0}; do
  PMK_TMA_CFG=$cfg ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --print-kernel-base demangled -k "regex:march_tma" -c 60 --csv \
    --log-file gpurun_out/ab_$cfg.csv python bench.py --case c5_c --steps 1 --warmup 0 \
    --e2e-steps 0 --no-cpu-baseline --no-profile > gpurun_out/ab_$cfg.log 2>&1
  echo "cfg $cfg"
  python tools/ncu_summary.py gpurun_out/ab_$cfg.csv | grep -E "march_(mvr|imv)\[2d\] \| \[(4.29|2.15)"
done
