#!/bin/bash
# A/B a runtime knob on the GPU box: alternate bench.py runs under two
# environment settings (device-timed ms_per_step of each run).
#   bash tools/ab_env.sh "PMK_PJ=0" "PMK_PJ=1" [rounds] [case]
mkdir -p gpurun_out
A=$1; B=$2; N=${3:-2}; CASE=${4:-c5_c}
for r in $(seq 1 $N); do
  for cfg in "$A" "$B"; do
    out=$(env $cfg python bench.py --case $CASE --steps 5 --warmup 3 --e2e-steps 0 \
          --no-cpu-baseline --no-profile --no-extra 2>/dev/null | tail -1)
    echo "$cfg $(echo "$out" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["iterations"], d["clocks"]["sm_mhz"])')"
  done
done
