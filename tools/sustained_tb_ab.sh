#!/bin/bash
# Sustained headline A/B at a given fused depth: TB=<d> bash tools/sustained_tb_ab.sh v1 v2 ...
for r in 1 2; do
  for v in "$@"; do
    L=build/qv_$v/libssam_b200.so; [ "$v" = main ] && L=paper_1907_06154_b200/libssam_b200.so
    SSAM_B200_LIB=$L timeout 300 python bench.py --steps 10 --warmup 3 --tb ${TB:-2} --no-e2e --no-cpu --no-suite --no-parity --no-traffic > /tmp/b.json 2>/dev/null
    python -c "import json,sys; d=json.load(open('/tmp/b.json')); print(sys.argv[1], 'tb', sys.argv[2], d['value'], d['roofline']['frac'], d['roofline']['mean_launch_ms'], d['clocks']['sm_mhz'])" $v ${TB:-2}
  done
done
