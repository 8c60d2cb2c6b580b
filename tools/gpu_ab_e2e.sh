#!/bin/bash
# One gpurun call: the C1 e2e number (pinned host -> library -> pinned host) per cache-slack setting, alternated.
mkdir -p gpurun_out
for rep in 1 2; do
  for sl in 16 64; do
    DZ_BENCH_SLACK_CHUNKS=$sl timeout 300 python bench.py --no-cpu-baseline --no-secondary --steps 50 ${BENCH_ARGS:-} > gpurun_out/e2e_ab.json 2> gpurun_out/e2e_ab.err
    echo "[$rep slack $sl] $(python -c "import json; d=json.load(open('gpurun_out/e2e_ab.json')); print(d['value'], d['e2e']['value'])")"
  done
done
