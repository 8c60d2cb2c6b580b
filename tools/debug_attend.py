"""Quick GPU triage: run attend on several shapes, each in a subprocess with a timeout."""
import os, subprocess, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))

CASES = {
    "h1_c1": dict(heads=1), "h4_c1": dict(heads=4), "h24_c1": dict(heads=24), "h25_c1": dict(heads=25),
    "h40_c1": dict(heads=40), "h40_c0chunks": dict(heads=40, cached_chunks=0),
}

def one(name):
    import numpy as np, torch, synth
    from helpers import GpuRun, errors
    kw = CASES[name]
    w = synth.scaled(synth.workload("C1"), **kw)
    run = GpuRun(w, capacity=max(w.cache_tokens, 1))
    run.fill(); torch.cuda.synchronize()
    import paper_2602_15922_b200 as dz
    t = time.time(); out = run.attend(); torch.cuda.synchronize(); dt = time.time() - t
    wd = dz.watchdog()
    if wd[0]:
        print(name, "WATCHDOG block", wd[1], "warp", wd[2], "bar_off", wd[3] - wd[6], "parity", wd[4], "sm", wd[5], flush=True)
    out = out.cpu().double().numpy()[0]
    hs = sorted({0, w.heads - 1})
    rows = np.arange(0, w.chunk_tokens, 11)
    for h in hs:
        want = run.oracle_out(heads=(h, h + 1), rows=rows)
        print(name, "head", h, "err", errors(out[rows, h:h + 1], want), "t", dt, flush=True)

if __name__ == "__main__":
    if len(sys.argv) > 1:
        one(sys.argv[1]); sys.exit(0)
    for name in CASES:
        try:
            r = subprocess.run([sys.executable, __file__, name], timeout=90, capture_output=True, text=True)
            print(r.stdout.strip()); print(r.stderr.strip()[-1500:]) if r.returncode else None
            print(name, "rc", r.returncode, flush=True)
        except subprocess.TimeoutExpired:
            print(name, "TIMEOUT", flush=True)
