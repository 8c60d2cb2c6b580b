"""One-line summary of a bench.py JSON line."""
import json
import sys

try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    r, k = d["roofline"], d["kernels"]
    print(f"value {d['value']:.1f} TF/s step-median {d['step_ms']['median'] * 1e3:.1f} us ({100 * d['pct_peak']:.1f}% peak) ms/step {d['ms_per_step']:.4f} | attn "
          f"{r['k2_ms']['median'] * 1e3:.1f} us {r['achieved']:.1f} TF/s frac {r['frac']:.3f} @ {r.get('k2_sm_ghz') or 0:.3f} GHz "
          f"(per clock {r.get('frac_per_clock_k2') or 0:.3f}) | prologue "
          f"{k['prologue_ms']['median'] * 1e3:.1f} us {k['prologue_gbs']:.0f} GB/s | append {k['append_ms']['median'] * 1e3:.1f} us "
          f"{k['append_gbs'] or 0:.0f} GB/s | e2e {d['e2e']['value'] if d.get('e2e') else None} | clocks {d['clocks']}")
except Exception as e:  # noqa: BLE001
    print("bench parse failed:", e)
