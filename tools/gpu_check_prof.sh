#!/bin/bash
# gpu_check.sh + one ncu --set full capture of K2 on the short bench command.
bash tools/gpu_check.sh
SHORT="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0"
timeout 300 $SHORT > gpurun_out/short.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 4 -c 1 -o gpurun_out/attn_full -f $SHORT > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
