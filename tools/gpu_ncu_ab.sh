#!/bin/bash
# ncu --set full of K2 for libdz_old.so and libdz.so (short bench command, each run clean first)
mkdir -p gpurun_out
SHORT="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0"
for L in old new; do
  F=paper_2602_15922_b200/libdz.so; [ $L = old ] && F=paper_2602_15922_b200/libdz_old.so
  export DZ_LIB_PATH=$PWD/$F
  timeout 300 $SHORT > gpurun_out/short_$L.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 4 -c 1 -o gpurun_out/attn_$L -f $SHORT > gpurun_out/ncu_$L.log 2>&1; echo "ncu $L rc=$?"
done
