#!/bin/bash
# A/B of 2D star stencils (tools/st2d_time.py) across builds, two passes:
#   bash tools/st2d_star64_ab.sh lib1.so lib2.so ...
# (variants: make qvariant VAR=x VSRC=stencil2d VFLAGS="-D...")
for rep in 1 2; do
  for L in "$@"; do
    echo -n "$L "
    SSAM_B200_LIB=$L timeout 120 python tools/st2d_time.py 2d17pt 2d21pt 2ds25pt 2>&1 | tail -1
  done
done
