#!/bin/bash
# One gpurun call: GPU tests (PYTEST_ARGS), then one short bench line per environment setting
# given as arguments ("NAME=VALUE" or "-" for none), summarised by tools/bench_brief.py.
mkdir -p gpurun_out
if [ -n "${PYTEST_ARGS:-}" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q $PYTEST_ARGS > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
  tail -3 gpurun_out/pytest_gpu.log
fi
i=0
for setting in "$@"; do
  i=$((i+1))
  if [ "$setting" = "-" ]; then envs=""; else envs="$setting"; fi
  env $envs timeout 300 python bench.py --no-cpu-baseline --steps 100 --e2e-steps 10 ${BENCH_ARGS:-} > gpurun_out/ab_$i.json 2> gpurun_out/ab_$i.err
  echo "[$setting] rc=$? $(python tools/bench_brief.py gpurun_out/ab_$i.json 2>&1)"
done
