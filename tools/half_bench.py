"""K2 cost of a half unit (<= 128 query rows, M = 128 pair MMAs) against a full unit (256 rows).

Each case is a Wan-shaped layer (40 heads x 128) with ~6.7 K keys and a chunk of nq tokens, so every
query group is a half unit (nq = 128), or a full one (nq = 256); DZ_DEBUG_KERNEL=2 runs the nq = 128 case
as padded M = 256 units instead.  Prints the median K2 time (library events) per case.
    DZ_LIB_PATH=... python tools/half_bench.py
"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np, torch, synth
import paper_2602_15922_b200 as dz
from helpers import GpuRun

B = int(os.environ.get("BATCH", "4"))  # 160 units over 74 pairs: mostly whole units
cases = {
    "nq128": synth.scaled(synth.workload("C1"), batch=B, frames=1, grid_h=4, grid_w=8, views=1, actions=96,
                          cached_chunks=52),
    "nq256": synth.scaled(synth.workload("C1"), batch=B, frames=1, grid_h=4, grid_w=8, views=1, actions=224,
                          cached_chunks=26),
}
for name, w in cases.items():
    run = GpuRun(w, flags=dz.FLAG_PROFILE if hasattr(dz, "FLAG_PROFILE") else 0)
    run.fill()
    run.cache.profile_enable(True)
    t = []
    for i in range(40):
        run.attend()
        torch.cuda.synchronize()
        if i >= 5:
            t.append(run.cache.profile_last()["attention"])
    units = run.cache.attention_units(w.chunk_tokens)
    steps = (w.kv_tokens + 127) // 128
    med = float(np.median(t)) * 1e3
    print(f"{name}: nq {w.chunk_tokens} kv {w.kv_tokens} units {units} steps/unit {steps}: K2 {med:.1f} us, "
          f"{med * 1e3 / (units * steps / 74):.1f} ns per unit-step per pair", flush=True)
    run.cache.close()
