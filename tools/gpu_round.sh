#!/bin/bash
# One gpurun call: tests, bench, launch list, ncu captures.  Output -> gpurun_out/
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt
free -g >> gpurun_out/gpu.txt; nproc >> gpurun_out/gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1
timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --iters 10 --no-e2e --no-cpu --no-suite --no-parity --no-traffic > gpurun_out/launches_bench.json 2>&1
for spec in ${NCU_SPECS}; do
  tag=$(echo $spec | tr ':' '_')
  args=$(echo $spec | tr ':' ' ')
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:ssam -s 1 -c 1 -o gpurun_out/prof_$tag python tools/prof_one.py $args > gpurun_out/prof_$tag.log 2>&1
done
ls -la gpurun_out
