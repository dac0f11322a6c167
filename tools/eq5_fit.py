"""Fit the paper's step-time model, Eq. 5 (T_batch constant,
T_sync ~ log N), t_step(N) = A + B * log2(N), to the measured bench lines under
profiles/ (N = 1, 2, 4).  Prints A, B and R^2 per workload."""
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
RUNS = {
    "C2-jet": ["r01_c2_bench_final.json", "r01_c2_bench_n2_final.json", "r01_c2_bench_n4_final.json"],
    "C3-imdb": ["r01_c3_bench_final.json", None, "r01_c3_bench_n4_final.json"],
    "C4-stacked": ["r01_c4_bench_final.json", "r01_c4_bench_n2.json", "r01_c4_bench_n4_final.json"],
}


def load(name):
    with open(os.path.join(ROOT, "profiles", name)) as f:
        line = [l for l in f if l.startswith("{")][-1]
    return json.loads(line)


def fit(xs, ys):
    n = len(xs)
    mx, my = sum(xs) / n, sum(ys) / n
    sxx = sum((x - mx) ** 2 for x in xs)
    B = sum((x - mx) * (y - my) for x, y in zip(xs, ys)) / sxx
    A = my - B * mx
    ss_res = sum((y - A - B * x) ** 2 for x, y in zip(xs, ys))
    ss_tot = sum((y - my) ** 2 for y in ys)
    return A, B, (1 - ss_res / ss_tot) if ss_tot > 0 else 1.0


out = {}
for wl, files in RUNS.items():
    pts = []
    for f in files:
        if f is None:
            continue
        d = load(f)
        pts.append((d["n_gpus"], d["ms_per_step"], d["value"]))
    xs = [math.log2(n) for n, _, _ in pts]
    ys = [t for _, t, _ in pts]
    A, B, r2 = fit(xs, ys)
    out[wl] = {"points": [{"n": n, "ms_per_step": round(t, 4), "samples_per_s": round(v)} for n, t, v in pts],
               "A_ms": round(A, 4), "B_ms_per_doubling": round(B, 4), "R2": round(r2, 3)}
json.dump(out, sys.stdout, indent=1)
print()
