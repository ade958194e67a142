#!/bin/bash
# One `ncu --set full` capture per hot kernel of a c5_c solve (run on the GPU
# box): fine K-MVR, fine K-IMV, the coarsest sine transforms.
#   bash tools/ncu_full.sh <tag>
mkdir -p gpurun_out
T=${1:-r1}
run() {  # name regex skip
  ncu --set full --clock-control none --import-source on -k "regex:$2" --launch-skip $3 \
    --launch-count 1 -o gpurun_out/${T}_$1 -f python bench.py --case c5_c --steps 1 --warmup 0 \
    --e2e-steps 0 --no-cpu-baseline --no-profile --no-extra > gpurun_out/${T}_$1.log 2>&1
  echo "$1 rc $?"
}
run mvr_fine march_tma 0
run imv_fine march_tma 21
run dst_rows dst_rows 0
run dst_cols dst_cols 0
