#!/bin/bash
# A/B builds of the library on the GPU box (same box, alternating runs):
#   bash tools/ab_lib.sh "libpmk_b200_a.so libpmk_b200_b.so" [rounds] [case]
# (the default libpmk_b200.so always runs first in each round; variants are
# built with: make -C paper_2401_00228_b200/csrc VARIANT=name EXTRA=-D...)
mkdir -p gpurun_out
V=$1; N=${2:-2}; CASE=${3:-c5_c}
for r in $(seq 1 $N); do
  for lib in libpmk_b200.so $V; do
    out=$(PMK_LIB=paper_2401_00228_b200/$lib python bench.py --case $CASE --steps 5 --warmup 3 \
          --e2e-steps 0 --no-cpu-baseline --no-extra 2>/dev/null | tail -1)
    echo "$lib $(echo "$out" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); k=d["kernels"]; print(round(d["ms_per_step"],2), d["iterations"], d["clocks"]["sm_mhz"], "mvr", k["march_mvr"]["ms"], "imv", k["march_imv"]["ms"])')"
  done
done
