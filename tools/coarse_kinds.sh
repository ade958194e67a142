#!/bin/bash
# Coarsest kinds side by side on one box (CUDA events around the coarsest
# solve alone): the default choice vs PMK_COARSE_KIND forced.
#   bash tools/coarse_kinds.sh > gpurun_out/coarse_kinds.txt
for spec in "agg1_mid:pcr eig" "pcr_dec_mid:pcr eig" "c2_c:pcr" "c1:pcr" "line_mid:line" "line_dec_mid:line" \
            "c3_c:line" "ttts_mid:line"; do
  case=${spec%%:*}
  python tools/coarse_probe.py $case 20
  for k in ${spec#*:}; do PMK_COARSE_KIND=$k python tools/coarse_probe.py $case 20; done
done
