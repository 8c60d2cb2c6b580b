#!/bin/bash
# One gpurun iteration: GPU tests, bench line, K2 trace, and an ncu --set full capture of
# the kernel matching $NCU_K (default: prologue) on the short bench command.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
SHORT="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0"
timeout 300 python bench.py --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python tools/bench_brief.py gpurun_out/bench.json
timeout 120 python tools/trace_c.py C1 > gpurun_out/trace.txt 2>&1; head -12 gpurun_out/trace.txt
if [ -n "${NCU_K:-}" ]; then
timeout 300 $SHORT > gpurun_out/short.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${NCU_K} -s ${NCU_S:-2} -c ${NCU_C:-2} -o gpurun_out/prof -f $SHORT > gpurun_out/ncu_full.log 2>&1; echo "ncu rc=$?"
fi
