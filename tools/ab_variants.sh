#!/bin/bash
# Bench A/B of library variants paper_2602_15922_b200/libdz*.so (attention / prologue / append times).
for L in ${LIBS:-paper_2602_15922_b200/libdz.so}; do
echo -n "$L: "; DZ_LIB_PATH=$PWD/$L timeout 200 python bench.py --no-cpu-baseline --e2e-steps 0 --steps 100 > /tmp/b.json 2>/dev/null; python tools/bench_brief.py /tmp/b.json
done
