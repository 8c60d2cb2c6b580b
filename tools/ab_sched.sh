#!/bin/bash
for i in 1 2; do
for S in sk rr; do
echo -n "$S: "; if [ $S = rr ]; then export DZ_SCHED_RR=1; else unset DZ_SCHED_RR; fi
timeout 200 python bench.py --no-cpu-baseline --e2e-steps 0 --steps 100 > /tmp/b.json 2>/dev/null; python tools/bench_brief.py /tmp/b.json | cut -c1-120
done; done
