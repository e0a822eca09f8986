"""Small workloads for compute-sanitizer: the cluster-resident solver (f64 and
mixed, R = 1, a 16-CTA and a 10-CTA cluster, overflow re-solve), pose LM, triangulation
and matching."""
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [REPO, os.path.join(REPO, "src"), os.path.join(REPO, "tests")]


def main():
    import torch
    from gpu_helpers import run_device
    from paper_2506_05558_b200.synth import make_batch
    b = make_batch(3, n_cams=8, K=800, seed=4)
    probs = [b.problem(i) for i in range(3)]
    for prec in ("f64", "mixed"):
        run_device(probs, dict(max_iters=8), prec, "auto")
    big = make_batch(1, n_cams=6, K=9000, seed=5).problem(0)
    run_device([big], dict(max_iters=4), "f64", "auto")      # cluster of CTAs
    os.environ["MBA_V4_R"] = "10"                             # non-power-of-two cluster
    run_device([big], dict(max_iters=4), "f64", "auto")
    run_device([big], dict(max_iters=4), "mixed", "auto")
    del os.environ["MBA_V4_R"]
    os.environ["MBA_V4_ARENA_CAP"] = "20000"
    run_device(probs[:1], dict(max_iters=4), "f64", "auto")  # overflow -> CTA kernel
    del os.environ["MBA_V4_ARENA_CAP"]
    from gsrecon import miniba as M
    from gsrecon.scene import CameraIntrinsics
    z = np.load(os.path.join(REPO, "tests", "golden", "triangulate.npz"))
    intr = CameraIntrinsics(float(z["focal"]), float(z["cx"]), float(z["cy"]), 640, 480)
    M.triangulate_batch(z["R"], z["t"], z["cam"], z["uv"], z["obs_off"][:101], intr)
    m = np.load(os.path.join(REPO, "tests", "golden", "match.npz"))
    off = m["desc_off"]
    M.match_batch([m["desc"][off[f]:off[f + 1]] for f in range(3)], [(0, 1), (1, 2)])
    torch.cuda.synchronize()
    print("sanitize workload done")


if __name__ == "__main__":
    main()
