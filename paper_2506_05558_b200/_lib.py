"""ctypes binding of libminiba.so (include/miniba.h).

PyTorch is used only for device memory and the current CUDA stream. There is
no CPU fallback: every entry point raises if the library or a CUDA device is
missing.
"""
from __future__ import annotations

import ctypes as ct
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MBA_LIB", os.path.join(HERE, "libminiba.so"))

MBA_OK, MBA_ERR_INVALID, MBA_ERR_TOO_LARGE, MBA_ERR_CUDA, MBA_ERR_EMPTY, MBA_ERR_NOT_PD = 0, -1, -2, -3, -4, -5
LOSS = {"huber": 0, "cauchy": 1}
PRECISION = {"f32": 0, "mixed": 0, "f64": 1}

_vp = ct.c_void_p


class MbaBatchDesc(ct.Structure):
    _fields_ = [("n_problems", ct.c_int32), ("max_cams", ct.c_int32), ("max_obs", ct.c_int64),
                ("max_points", ct.c_int64), ("max_pairs", ct.c_int64),
                ("max_track", ct.c_int32), ("reserved", ct.c_int32), ("cam_off", _vp), ("pt_off", _vp), ("obs_off", _vp),
                ("obs", _vp), ("obs_lo", _vp), ("fixed", _vp), ("cx", _vp), ("cy", _vp),
                ("flags", _vp)]


class MbaLmConfig(ct.Structure):
    _fields_ = [("lambda_init", ct.c_double), ("nu", ct.c_double), ("delta", ct.c_double),
                ("max_iters", ct.c_int32), ("loss", ct.c_int32), ("precision", ct.c_int32),
                ("ctas_per_problem", ct.c_int32), ("fail_iters_mask", ct.c_uint64)]


class MbaOutputs(ct.Structure):
    _fields_ = [(n, _vp) for n in ("R_in", "t_in", "focal_in", "points_in", "R_out", "t_out",
                                   "focal_out", "points_out", "costs", "lambdas", "accepted",
                                   "evals", "n_iters", "status", "final_stats")]


_lib = None


def lib():
    """Load libminiba.so; fail loudly (no fallback) when it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`"
                           " (the mini-BA has no CPU fallback)")
    L = ct.CDLL(LIB_PATH)
    i32, i64, d, sz = ct.c_int32, ct.c_int64, ct.c_double, ct.c_size_t
    L.mba_abi_version.restype = i32
    L.mba_workspace_bytes.restype = sz
    L.mba_workspace_bytes.argtypes = [ct.POINTER(MbaBatchDesc), ct.POINTER(MbaLmConfig)]
    L.mba_solve.restype = i32
    L.mba_solve_plan.restype = i32
    L.mba_solve_plan.argtypes = [ct.POINTER(MbaBatchDesc), ct.POINTER(MbaLmConfig)]
    L.mba_match_pairs.restype = i32
    L.mba_match_pairs.argtypes = [i32, _vp, _vp, i32, _vp, _vp, _vp, i64, d, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                                  i64, i64, _vp, sz, _vp]
    L.mba_match_workspace_bytes.restype = sz
    L.mba_match_workspace_bytes.argtypes = [i64, i64, i64]
    L.mba_triangulate.restype = i32
    L.mba_triangulate.argtypes = [i32, _vp, _vp, _vp, i32, _vp, _vp, d, d, d, d, d, i32, _vp, _vp, _vp, _vp]
    L.mba_solve_launches.restype = i32
    L.mba_solve_launches.argtypes = [ct.POINTER(MbaBatchDesc), ct.POINTER(MbaLmConfig)]
    L.mba_solve.argtypes = [ct.POINTER(MbaBatchDesc), ct.POINTER(MbaLmConfig),
                            ct.POINTER(MbaOutputs), _vp, sz, _vp]
    L.mba_residuals.restype = i32
    L.mba_residuals.argtypes = [i64, _vp, _vp, d, d, d, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]
    L.mba_robust.restype = i32
    L.mba_robust.argtypes = [i64, _vp, d, i32, _vp, _vp, _vp]
    L.mba_blocks.restype = i32
    L.mba_blocks.argtypes = [i64, _vp, _vp, d, _vp, _vp, _vp, _vp, _vp, _vp, _vp]
    L.mba_assemble.restype = i32
    L.mba_assemble.argtypes = [i64, i32, i32, i64, _vp, _vp, i32, i32, _vp, _vp, _vp, _vp, _vp,
                               _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]
    L.mba_solve_step_scratch_bytes.restype = sz
    L.mba_solve_step_scratch_bytes.argtypes = [i32, i64, i32]
    L.mba_solve_step.restype = i32
    L.mba_solve_step.argtypes = [i32, i64, _vp, _vp, _vp, _vp, _vp, d, i32, _vp, _vp, _vp, _vp]
    L.mba_pose_lm.restype = i32
    L.mba_pose_lm.argtypes = [i32, i32, _vp, _vp, d, d, d, i32, d, d, d, _vp, _vp, _vp, i32, _vp,
                              _vp, d, _vp, _vp, _vp]
    L.mba_pack_obs_workspace_bytes.restype = sz
    L.mba_pack_obs_workspace_bytes.argtypes = [i64]
    L.mba_pack_obs.restype = i32
    L.mba_pack_obs.argtypes = [i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, sz, _vp]
    L.mba_compact_traces.restype = i32
    L.mba_compact_traces.argtypes = [i32, i32] + [_vp] * 10 + [_vp]
    L.mba_bootstrap_workspace_bytes.restype = sz
    L.mba_bootstrap_workspace_bytes.argtypes = [ct.POINTER(MbaBatchDesc), ct.POINTER(MbaLmConfig)]
    L.mba_bootstrap_schedule.restype = i32
    L.mba_bootstrap_schedule.argtypes = [ct.POINTER(MbaBatchDesc), ct.POINTER(MbaLmConfig),
                                         ct.POINTER(MbaLmConfig), d, ct.POINTER(MbaOutputs),
                                         ct.POINTER(MbaOutputs), _vp, _vp, _vp, _vp, _vp, _vp, _vp, sz, _vp]
    if L.mba_abi_version() != 1:
        raise RuntimeError("libminiba ABI version mismatch")
    _lib = L
    return L


EXPORTED = ("mba_abi_version", "mba_workspace_bytes", "mba_solve", "mba_solve_plan", "mba_solve_launches", "mba_residuals", "mba_robust",
            "mba_blocks", "mba_assemble", "mba_solve_step_scratch_bytes", "mba_solve_step",
            "mba_pose_lm", "mba_triangulate", "mba_match_pairs", "mba_match_workspace_bytes", "mba_pack_obs_workspace_bytes",
            "mba_pack_obs", "mba_bootstrap_workspace_bytes", "mba_bootstrap_schedule",
            "mba_compact_traces")


def check(rc, what):
    if rc == MBA_OK:
        return
    if rc in (MBA_ERR_INVALID, MBA_ERR_EMPTY):
        raise ValueError(f"{what}: invalid input (status {rc})")
    if rc == MBA_ERR_NOT_PD:
        raise np.linalg.LinAlgError(f"{what}: matrix is not positive definite")
    if rc == MBA_ERR_TOO_LARGE:
        raise ValueError(f"{what}: problem exceeds the device plan (too many cameras)")
    raise RuntimeError(f"{what}: CUDA failure (status {rc})")


def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("mini-BA needs a CUDA device (sm_100a); there is no CPU fallback")
    return torch


def stream_ptr():
    torch = torch_cuda()
    return _vp(torch.cuda.current_stream().cuda_stream)


def ptr(t):
    return None if t is None else _vp(t.data_ptr())
