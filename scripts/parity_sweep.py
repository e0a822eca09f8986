"""Parity sweep: solve the first N problems of a BASELINE workload on the
device and with the CPU oracle, and report how many meet the SURVEY 8c rule
(identical accepted/evals/lambda through i*, final cost rel <= 1e-4, rotation
<= 1e-4 rad, translation rel <= 1e-4).

    python scripts/parity_sweep.py --config 4 --problems 256 --precision mixed
"""
import argparse
import json
import os
import sys
from concurrent.futures import ProcessPoolExecutor

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [REPO, os.path.join(REPO, "src"), os.path.join(REPO, "tests")]


def _oracle(args):
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    sys.path[:0] = [REPO]
    from oracle import miniba_oracle as O
    p, max_iters, loss = args
    info = O.lm(p, max_iters=max_iters, loss=loss)
    return info, p["R"], p["t"], p["focal"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--problems", type=int, default=256)
    ap.add_argument("--precision", default="mixed")
    ap.add_argument("--kernel", default="auto")
    a = ap.parse_args()
    from gpu_helpers import rot_err, run_device
    from oracle import miniba_oracle as O
    from paper_2506_05558_b200.synth import CONFIGS, make_batch
    c = CONFIGS[a.config]
    n = min(a.problems, c["n_problems"])
    b = make_batch(n, n_cams=c["n_cams"], K=c["K"], outlier_frac=c.get("outlier_frac", 0.0))
    probs = [b.problem(i) for i in range(n)]
    dev = run_device(probs, dict(max_iters=c["max_iters"], loss=c["loss"]), a.precision, a.kernel)
    with ProcessPoolExecutor(len(os.sched_getaffinity(0))) as ex:
        refs = list(ex.map(_oracle, [(b.problem(i), c["max_iters"], c["loss"]) for i in range(n)]))
    stats = dict(trace=0, cost=0, rot=0, trans=0, all=0)
    worst = dict(cost=0.0, rot=0.0, trans=0.0)
    for d, (ref, R, t, f) in zip(dev, refs):
        i_star = O.plateau_index(ref["costs"])
        m = i_star + 1
        tr = (len(d["accepted"]) >= m and np.array_equal(d["accepted"][:m], ref["accepted"][:m])
              and np.array_equal(d["evals"][:m], ref["evals"][:m]))
        cr = abs(d["costs"][-1] - ref["costs"][-1]) / abs(ref["costs"][-1])
        rr = max(rot_err(d["R"][k], R[k]) for k in range(len(R)))
        tt = np.abs(d["t"] - t).max() / np.linalg.norm(t, axis=1).max()
        ok = [tr, cr <= 1e-4, rr <= 1e-4, tt <= 1e-4]
        for k, v in zip(("trace", "cost", "rot", "trans"), ok):
            stats[k] += int(v)
        stats["all"] += int(all(ok))
        worst["cost"] = max(worst["cost"], cr)
        worst["rot"] = max(worst["rot"], rr)
        worst["trans"] = max(worst["trans"], tt)
    print(json.dumps(dict(config=a.config, problems=n, precision=a.precision, kernel=a.kernel,
                          pass_counts=stats, worst=worst)))


if __name__ == "__main__":
    main()
