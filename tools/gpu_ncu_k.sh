#!/bin/bash
# ncu --set full of kernels matching $K (launches $S.. count $C) on the short bench command (run clean first).
mkdir -p gpurun_out
SHORT="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0"
timeout 300 $SHORT > gpurun_out/short.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${K} -s ${S:-2} -c ${C:-2} -o gpurun_out/prof_${K} -f $SHORT > gpurun_out/ncu_${K}.log 2>&1; echo "ncu rc=$?"
