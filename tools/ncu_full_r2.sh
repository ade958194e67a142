#!/bin/bash
# Round-2 `ncu --set full` captures (one launch each, on the GPU box): the
# fine-level in-solver march kernels and coarsest sine transforms of a c5_c
# solve (tools/ncu_full.sh), the plain matvec on 16-row tiles, and the PCR /
# LINE coarsest chains.
#   bash tools/ncu_full_r2.sh <tag>
T=${1:-r2f}
bash tools/ncu_full.sh $T
cap() {  # name regex command...
  local name=$1 rx=$2; shift 2
  ncu --set full --clock-control none --import-source on -k "regex:$rx" --launch-skip 3 \
    --launch-count 1 -o gpurun_out/${T}_$name -f "$@" > gpurun_out/${T}_$name.log 2>&1
  echo "$name rc $?"
}
cap mv_tall march_tma python tools/mv_probe.py c5_c 3
cap line_chain line_chain python tools/coarse_probe.py line_mid 5
cap pcr_chain pcr_chain python tools/coarse_probe.py pcr_dec_mid 5
