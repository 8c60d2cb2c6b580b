#!/bin/bash
for f in 0 4 7; do echo -n "DZ_DEBUG_KERNEL=$f: "; DZ_DEBUG_KERNEL=$f timeout 120 python bench.py --no-cpu-baseline --e2e-steps 0 --steps 50 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['roofline']['attn_ms_mean']*1e3,1),'us', round(d['roofline']['achieved'],1),'TF/s')"; done
