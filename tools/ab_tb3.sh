# A/B of the fused Tb=2 3D kernel: LIBS="a.so b.so" bash tools/ab_tb3.sh
for i in 1 2; do
for L in ${LIBS}; do
  echo "== $L"
  SSAM_B200_LIB=$L timeout 100 python tools/tb3d_time.py 514 f32
  SSAM_B200_LIB=$L timeout 100 python tools/tb3d_time.py 130 f64
  SSAM_B200_LIB=$L timeout 100 python tools/run3d_time.py 3d7pt f32 512 20
  SSAM_B200_LIB=$L timeout 100 python tools/run3d_time.py 3d7pt f64 512 20
done
done
