#!/bin/bash
# One gpurun call: C3 denoise graph lines per library (value and median step), alternating, twice.
mkdir -p gpurun_out
for i in 1 2; do for lib in "$@"; do
  DZ_LIB_PATH=$PWD/paper_2602_15922_b200/$lib timeout 300 python bench.py --workload C3 --mode denoise --graph --no-cpu-baseline --e2e-steps 0 --steps 40 --no-secondary > gpurun_out/dn.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/dn.json').read().strip().splitlines()[0]); print('[$lib]', round(d['value'],1), d['unit'], 'median step', round(d['step_ms']['median']*1e3,1), 'us')"
done; done
