"""Refit the B200 weights w1..w7 of Alg. 2 (§6.1) from measured
schedule sweeps (profiles/sweep_<round>_<workload>.txt, written by tools/sweep.py on a B200).

For every measured configuration the seven B200-mode terms are recomputed on the host (pmg_schedule with that
manual configuration; ptxas register counts from an NVRTC compile, as the selector's probe does).  A weight
vector is scored by how slow the configuration it would pick is: loss = mean over workloads of
log(t[argmin cost] / t[best measured]).  The paper fits by leave-one-out cross-validation over benchmarks
(P:1158-1162); this script reports the LOOCV loss of the fitting procedure and the weights fitted on all
workloads.

    python tools/fit_weights.py --round r01 harris unsharp blur
"""
import argparse
import json
import math
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import paper_1909_07190_b200 as pmg  # noqa: E402
import pmg_inputs as PI  # noqa: E402

TERMS = ["txsPerPoint", "1-occupancy", "memTime/computeTime", "unallocatedShMem", "unusedReg", "fracOverlap",
         "extraTBs"]


def term_vector(cost):
    r = cost["memTime"] / cost["computeTime"] if cost["computeTime"] > 0 else 0.0
    return [cost["txsPerPoint"], 1 - cost["occupancy"], r, cost["unallocatedShMem"], cost["unusedReg"],
            cost["fracOverlap"], cost["extraTBs"]]


def load(round_, name):
    wl = PI.WORKLOADS[name]
    pipe = pmg.Pipeline(wl.text)
    spec = pmg.gpu_spec("b200")
    X, t, specs = [], [], []
    for line in open(ROOT / "profiles" / f"sweep_{round_}_{name}.txt"):
        if not line.startswith("{"):
            continue
        r = json.loads(line)
        if "ms" not in r or r["spec"] == "auto":
            continue
        kv = {k: int(v) for k, v in (x.split("=") for x in r["spec"].split(","))}
        s = pipe.schedule(wl.params, spec=spec, opts=pmg.sched_opts(**kv, probe=True))
        if len(s["groups"]) != 1:
            continue
        X.append(term_vector(s["groups"][0]["cost"]))
        t.append(r["ms"])
        specs.append(r["spec"])
    return np.array(X), np.array(t), specs


def loss(w, data):
    out = []
    for X, t, _ in data:
        c = X @ w
        out.append(math.log(t[int(np.argmin(c))] / t.min()))
    return float(np.mean(out))


def fit(data, iters=4000, seed=0):
    rng = np.random.default_rng(seed)
    best_w, best_l = None, float("inf")
    base = np.array([50, 0.5, 60, 10, 2, 100, 1], dtype=float)      # the V100 row (Table 3)
    for i in range(iters):
        if best_w is None or i < iters // 2:
            w = base * np.exp(rng.uniform(-4, 4, 7)) * (rng.random(7) > 0.25)
        else:
            w = best_w * np.exp(rng.normal(0, 0.5, 7)) * (rng.random(7) > 0.1)
        l_ = loss(w, data)
        # ties: prefer weights closer to the paper's row (smaller log-distance)
        if l_ < best_l - 1e-12:
            best_w, best_l = w, l_
    return best_w, best_l


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--round", default="r01")
    ap.add_argument("workloads", nargs="+")
    a = ap.parse_args()
    data = [load(a.round, n) for n in a.workloads]
    v100 = np.array([50, 0.5, 60, 10, 2, 100, 1], dtype=float)
    print("V100 weights: loss", round(loss(v100, data), 4), "per workload",
          [round(loss(v100, [d]), 4) for d in data])
    if len(data) > 1:
        cv = []
        for i in range(len(data)):
            w, _ = fit([d for j, d in enumerate(data) if j != i], seed=i)
            cv.append(loss(w, [data[i]]))
        print("LOOCV held-out losses", [round(x, 4) for x in cv], "mean", round(float(np.mean(cv)), 4))
    w, l_ = fit(data)
    print("fitted on all: loss", round(l_, 4), "weights", [float(f"{x:.4g}") for x in w])
    for (X, t, specs), n in zip(data, a.workloads):
        i = int(np.argmin(X @ w))
        print(f"  {n}: picks {specs[i]} {t[i]} ms (best {t.min()} ms)")


if __name__ == "__main__":
    main()
