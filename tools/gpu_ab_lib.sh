#!/bin/bash
# One gpurun call: a short bench line per "LIB[:ENV=VAL...]" argument (LIB under paper_2602_15922_b200/).
mkdir -p gpurun_out
i=0
for spec in "$@"; do
  i=$((i+1))
  lib=${spec%%:*}; envs=""; [ "$spec" != "$lib" ] && envs=$(echo "${spec#*:}" | tr ',' ' ')
  env DZ_LIB_PATH=$PWD/paper_2602_15922_b200/$lib $envs timeout 200 python bench.py --no-cpu-baseline --e2e-steps 0 --steps ${STEPS:-100} --no-secondary ${BENCH_ARGS:-} > gpurun_out/abl_$i.json 2> gpurun_out/abl_$i.err
  echo "[$spec] $(python tools/bench_brief.py gpurun_out/abl_$i.json 2>&1 | cut -c1-150)"
done
