#!/bin/bash
# One gpurun call: short bench lines of bench.py per BENCH_ARGS variant ("a|b|c", '_' = no flags), twice each.
mkdir -p gpurun_out
IFS='|' read -ra V <<< "${VARIANTS:-_}"
for i in 1 2; do
for a in "${V[@]}"; do
  [ "$a" = "_" ] && a=""
  timeout 200 python bench.py --no-cpu-baseline --e2e-steps 0 --steps ${STEPS:-100} --no-secondary $a > gpurun_out/ab.json 2> gpurun_out/ab.err
  echo "[$a] $(python tools/bench_brief.py gpurun_out/ab.json 2>&1 | cut -c1-150)"
done; done
