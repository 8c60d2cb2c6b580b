#!/bin/bash
# One gpurun call: the secondary bench lines (C2, C4 at 1 GPU, C3 denoise eager / graph) into gpurun_out/.
mkdir -p gpurun_out
run() { name=$1; shift; timeout 600 python bench.py --no-cpu-baseline --steps ${STEPS:-50} "$@" > gpurun_out/bench_$name.json 2> gpurun_out/bench_$name.err; echo "[$name] rc=$? $(python tools/bench_brief.py gpurun_out/bench_$name.json | cut -c1-190)"; }
run c3_denoise --workload C3 --mode denoise
run c3_denoise_graph --workload C3 --mode denoise --graph
run c2 --workload C2
run c4 --workload C4 --e2e-steps 5
run c3_chunk --workload C3
run tf --mode tf --steps 30
