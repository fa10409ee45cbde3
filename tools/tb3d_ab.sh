# A/B of the fused Tb=2 3D kernel across library variants: LIBS="path ..." (empty = default)
for lib in ${LIBS:-""}; do
  [ "$lib" = "default" ] && lib=""
  echo "== lib=${lib:-default}"
  SSAM_B200_LIB=$lib timeout 100 python tools/tb3d_check.py 512 512 512 2>&1 | grep 3d7pt
  SSAM_B200_LIB=$lib timeout 60 python tools/tb3d_time.py
done
