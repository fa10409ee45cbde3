#!/bin/bash
# z-segment / CTA-shape sweep for the 3D stencils at the slab size
for st in 3d7pt poisson 3d27pt 3d13pt; do
  for z in 16 24 32 48 64; do SSAM_B200_3D_ZSEG=$z python tools/perf_slab.py $st; done
  for cfg in "1 4" "2 4" "1 8" "2 8"; do set -- $cfg; echo -n "SX=$1 WPB=$2 "; SSAM_B200_3D_SX=$1 SSAM_B200_3D_WPB=$2 python tools/perf_slab.py $st; done
done
