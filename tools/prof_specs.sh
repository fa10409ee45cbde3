# ncu --set full of prof_one.py specs: SPECS="kind:arg:..." ; summaries + SASS mix only
mkdir -p gpurun_out
for sp in ${SPECS}; do
  t=pf_$(echo $sp | tr ':' '_')
  args=$(echo $sp | tr ':' ' ')
  timeout 300 ncu --set full --clock-control none --import-source on -k "regex:${KREGEX:-ssam}" -s ${SKIP:-1} -c ${COUNT:-1} -o /tmp/$t python tools/prof_one.py $args > gpurun_out/$t.log 2>&1
  python tools/ncu_summary.py /tmp/$t.ncu-rep > gpurun_out/$t.sum.txt
  ncu -i /tmp/$t.ncu-rep --page source --csv --print-source sass > /tmp/$t.sass.csv 2>/dev/null
  python tools/sass_mix.py /tmp/$t.sass.csv > gpurun_out/$t.mix.txt
  [ -n "$KEEP_SASS" ] && cp /tmp/$t.sass.csv gpurun_out/
done
