# ncu --set full of conv2d K in $KS under each SSAM_B200_CONV_FMA in $FS; summaries only
mkdir -p gpurun_out
# FS entries: FMA[:RY]
for K in ${KS:-7 20}; do for FR in ${FS:-0 3}; do
  F=${FR%%:*}; RY=0; [ "$FR" != "$F" ] && RY=${FR#*:}
  t=pc_${K}_${F}_${RY}
  SSAM_B200_CONV_RY=$RY SSAM_B200_CONV_FMA=$F timeout 300 ncu --set full --clock-control none --import-source on -k regex:ssam -s 1 -c 1 -o /tmp/$t python tools/prof_one.py conv $K > gpurun_out/$t.log 2>&1
  python tools/ncu_summary.py /tmp/$t.ncu-rep > gpurun_out/$t.sum.txt
  ncu -i /tmp/$t.ncu-rep --page source --csv --print-source sass > gpurun_out/$t.sass.csv 2>/dev/null
  ncu -i /tmp/$t.ncu-rep --page details --csv > gpurun_out/$t.details.csv 2>/dev/null
done; done
ls -la gpurun_out
