#!/bin/bash
# Serialised per-launch times of the march kernels of one c5_c solve under
# each PMK_IPC (work items per resident CTA), summarised per level.
#   bash tools/march_ipc.sh "8 4 2"      (on the GPU box, via gpurun)
mkdir -p gpurun_out
for q in ${1:-8}; do
  PMK_IPC=$q ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --print-kernel-base demangled -k "regex:march_tma" -c 420 --csv \
    --log-file gpurun_out/ipc_$q.csv python bench.py --case c5_c --steps 1 --warmup 0 \
    --e2e-steps 0 --no-cpu-baseline --no-profile --no-extra > gpurun_out/ipc_$q.log 2>&1
  echo "== PMK_IPC=$q"
  python tools/ncu_summary.py gpurun_out/ipc_$q.csv | grep -E "^\| march" | head -20
done
