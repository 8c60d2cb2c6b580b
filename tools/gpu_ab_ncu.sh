#!/bin/bash
# GPU tests, A/B bench of libdz_old.so vs libdz.so, then one ncu --set full of the new K2.
bash tools/gpu_ab_tests.sh
SHORT="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0"
timeout 300 $SHORT > gpurun_out/short.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 4 -c 1 -o gpurun_out/attn_new -f $SHORT > gpurun_out/ncu_new.log 2>&1; echo "ncu rc=$?"
