#!/bin/bash
# One gpurun call: round-2 ncu evidence of the current build: the launch list of a short bench (device
# time per launch) and one `ncu --set full` capture each of K2 (attn_fwd) and of the fused prologue.
mkdir -p gpurun_out
SHORT="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-secondary --e2e-steps 0"
timeout 300 $SHORT > gpurun_out/ev_short.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/ev_launches.csv $SHORT > gpurun_out/ev_ncu_launch.log 2>&1; echo "launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 4 -c 1 -o gpurun_out/ev_attn -f $SHORT > gpurun_out/ev_ncu_attn.log 2>&1; echo "ncu attn rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:prologue_dual2 -s 2 -c 1 -o gpurun_out/ev_pro -f $SHORT > gpurun_out/ev_ncu_pro.log 2>&1; echo "ncu prologue rc=$?"
python -c 'from paper_2602_15922_b200 import build as b; print(b.source_sha())' > gpurun_out/ev_libsha.txt
# NEXT-1 backward: launch list of one Wan-shape call and a full capture of the attention backward kernel
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev_bwd_launches.csv python tools/bwd_time.py 2 1344 40 > gpurun_out/ev_ncu_bwd_launch.log 2>&1; echo "bwd launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_bwd -s 2 -c 1 -o gpurun_out/ev_bwd -f python tools/bwd_time.py 2 1344 40 > gpurun_out/ev_ncu_bwd.log 2>&1; echo "ncu bwd rc=$?"
