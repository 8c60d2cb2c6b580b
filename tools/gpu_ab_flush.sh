#!/bin/bash
# One gpurun call: the C1 bench line under each L2-flush / cache-slack variant, alternated twice.
mkdir -p gpurun_out
for rep in 1 2; do
  for v in "--no-discard" "" "--no-flush" "SLACK=64" ; do
    args=$v; envs=""
    [ "$v" = "SLACK=64" ] && { args=""; envs="DZ_BENCH_SLACK_CHUNKS=64"; }
    env $envs timeout 200 python bench.py --no-cpu-baseline --e2e-steps 0 --no-secondary $args > gpurun_out/flush_ab.json 2> gpurun_out/flush_ab.err
    echo "[$rep ${v:-discard}] $(python tools/bench_brief.py gpurun_out/flush_ab.json 2>&1 | cut -c1-170)"
  done
done
