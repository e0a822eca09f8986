import glob
import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (REPO, os.path.join(REPO, "src")):
    if p not in sys.path:
        sys.path.insert(0, p)

GOLDEN = os.path.join(REPO, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built sm_100a library")
    config.addinivalue_line("markers", "slow: long-running")


def load_case(path):
    z = np.load(path, allow_pickle=False)
    d = {k: z[k] for k in z.files}
    prob = dict(R=d["R"].astype(np.float64), t=d["t"].astype(np.float64),
                focal=float(d["focal"]), cx=float(d["cx"]), cy=float(d["cy"]),
                points=d["points"].astype(np.float64), cam_idx=d["cam_idx"].astype(np.int64),
                pt_idx=d["pt_idx"].astype(np.int64), uv=d["uv"].astype(np.float64),
                fixed_cams=d["fixed_cams"].astype(bool),
                optimize_focal=bool(d["optimize_focal"]),
                optimize_points=bool(d["optimize_points"]))
    cfg = dict(lambda_init=float(d["lambda_init"]), nu=float(d["nu"]), delta=float(d["delta"]),
               max_iters=int(d["max_iters"]), loss=str(d["loss"]),
               fail_at=tuple(int(x) for x in d["fail_at"]))
    out = {k[4:]: d[k] for k in d if k.startswith("out_")}
    return prob, cfg, out


def golden_cases():
    return sorted(glob.glob(os.path.join(GOLDEN, "lm_*.npz")))


def golden_ids():
    return [os.path.basename(p)[3:-4] for p in golden_cases()]


@pytest.fixture
def cuda_ok():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return True
