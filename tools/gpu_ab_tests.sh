#!/bin/bash
# GPU tests, then A/B of libdz_old.so vs libdz.so on the bench (attention / prologue / append times).
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
bash tools/ab_libs.sh
