"""Small workloads for compute-sanitizer: the cluster-resident solver (f64 and
mixed, R = 1, a 16-CTA and a 10-CTA cluster, overflow re-solve), the
cooperative grid solver (12 cameras, f64 and mixed), the CTA solver on
20-camera problems (blocked LDL^T over 15 panels), the device pack / sort kernel through
lm_solve_batch (shuffled observations), the bootstrap schedule, pose LM,
triangulation and matching."""
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
    grid = make_batch(1, n_cams=12, K=6000, seed=6).problem(0)
    run_device([grid], dict(max_iters=3), "f64", "grid")     # cooperative grid kernel
    run_device([grid], dict(max_iters=3), "mixed", "grid")
    wide = make_batch(2, n_cams=20, K=3000, seed=7)               # CTA kernel, 19 free cameras:
    run_device([wide.problem(i) for i in range(2)], dict(max_iters=3), "f64", "auto")  # 15 LDL panels
    from gsrecon import miniba as M
    from gsrecon.config import CaptureConfig, LmConfig
    from gsrecon.scene import CameraIntrinsics
    # list path: native gather, device stable sort of shuffled observations
    ps = []
    for i in range(3):
        p = b.problem(i)
        perm = np.random.default_rng(i).permutation(len(p["uv"]))
        for k in ("cam_idx", "pt_idx", "uv"):
            p[k] = p[k][perm]
        ps.append(M.BaProblem(**p))
    M.lm_solve_batch(ps, LmConfig(max_iters=6))
    # bootstrap schedule (solve, filter, compaction, solve, gauge) on one window
    bz = np.load(os.path.join(REPO, "tests", "golden", "bootstrap_seed0.npz"))
    feats, o = [], 0
    for c in bz["counts"]:
        feats.append((bz["keypoints"][o:o + c], bz["ids"][o:o + c]))
        o += c

    def exact(fa, fb):
        _, ia, ib = np.intersect1d(fa[1], fb[1], assume_unique=True, return_indices=True)
        return ia.astype(np.int64), ib.astype(np.int64), np.zeros(len(ia))
    cfg = CaptureConfig()
    cfg.bootstrap_iters = 10
    bintr = CameraIntrinsics(float(bz["focal"]), float(bz["cx"]), float(bz["cy"]), int(bz["width"]),
                             int(bz["height"]))
    M.bootstrap_batch([feats], [bintr], cfg, matcher=exact)
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
