#!/bin/bash
# One gpurun call: bench line, ncu launch list of the same command, one full ncu capture of K2.
set -u
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv > $OUT/smi_before.csv
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
tail -c 3000 $OUT/bench.json
SHORT="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0"
timeout 300 $SHORT > $OUT/short.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv $SHORT > $OUT/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 4 -c 1 -o $OUT/attn_full -f $SHORT > $OUT/ncu_full.log 2>&1; echo "ncu full rc=$?"
tail -5 $OUT/ncu_full.log
# K1 prologue (attend: Q, K, V) and K4 append: one full capture each (launches 5 and 6 of the short run)
timeout 600 ncu --set full --clock-control none --import-source on -k regex:prologue -s 4 -c 2 -o $OUT/pro_full -f $SHORT > $OUT/ncu_pro.log 2>&1; echo "ncu prologue rc=$?"
timeout 300 python tools/copy_bench.py > $OUT/copy_bench.txt 2>&1; cat $OUT/copy_bench.txt
