#!/bin/bash
# K2 diagnostics in one gpurun call: pipeline trace of CTA 0 + ablations (DZ_DEBUG_KERNEL bits:
# 1 no K/V TMA, 2 no S TMEM loads, 4 no exponentials; results are garbage under these flags).
mkdir -p gpurun_out
timeout 120 python tools/trace_c.py C1 > gpurun_out/trace.txt 2>&1; echo "trace rc=$?"
cat gpurun_out/trace.txt | head -40
for f in 0 1 2 4 6 7; do echo -n "DZ_DEBUG_KERNEL=$f: "; DZ_DEBUG_KERNEL=$f timeout 120 python bench.py --no-cpu-baseline --e2e-steps 0 --steps 50 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['roofline']['attn_ms_mean']*1e3,1),'us', round(d['roofline']['achieved'],1),'TF/s')"; done
