mkdir -p gpurun_out
bash tools/sustained_ab.sh main dz5 dz7 di4 r14 > gpurun_out/sustained_ab3.txt 2>&1
for z in 256 512; do SSAM_B200_3D_TB_ZSEG=$z bash tools/sustained_ab.sh main | sed "s/^main/zseg$z/"; done >> gpurun_out/sustained_ab3.txt 2>&1
