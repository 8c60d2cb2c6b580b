#!/bin/bash
# One gpurun call: GPU parity tests (-x) then a bench line (no cpu baseline).
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --no-cpu-baseline ${BENCH_ARGS:-} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python - <<'PY'
import json
try:
    d = json.loads(open("gpurun_out/bench.json").read().strip().splitlines()[-1])
    r = d["roofline"]; k = d["kernels"]
    print(f"value {d['value']:.1f} TF/s ({100*d['pct_peak']:.1f}% peak) ms/step {d['ms_per_step']:.4f} | attn {r['attn_ms_mean']*1e3:.1f} us {r['achieved']:.1f} TF/s frac {r['frac']:.3f} | prologue {k['prologue_ms']*1e3:.1f} us {k['prologue_gbs']:.0f} GB/s | append {k['append_ms']*1e3:.1f} us | e2e {d['e2e']['value'] if d['e2e'] else None} | clocks {d['clocks']}")
except Exception as e:
    print("bench parse failed", e); print(open("gpurun_out/bench.err").read()[-2000:])
PY
