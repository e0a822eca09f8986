"""Camera geometry used around the mini-BA (drop-in for the parts of the
reference's gsrecon.scene that the mini-BA API exposes: scene.py:13-30,
126-273). Host-side helpers on tiny arrays; the solver itself re-implements
exp_so3 and projection on device (csrc/mba_common.cuh)."""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def skew(v) -> np.ndarray:
    a, b, c = (float(x) for x in v)
    return np.array([[0.0, -c, b], [c, 0.0, -a], [-b, a, 0.0]])


def exp_so3(w) -> np.ndarray:
    """Rodrigues map with the second-order series below 1e-12 rad."""
    w = np.asarray(w, dtype=np.float64)
    angle = float(np.linalg.norm(w))
    if angle < 1e-12:
        Wx = skew(w)
        return np.eye(3) + Wx + 0.5 * (Wx @ Wx)
    Kx = skew(w / angle)
    return np.eye(3) + np.sin(angle) * Kx + (1.0 - np.cos(angle)) * (Kx @ Kx)


def rotation6d_to_matrix(r6) -> np.ndarray:
    """Gram-Schmidt of the two stored columns; columns (c1, c2, c1 x c2)."""
    r6 = np.asarray(r6, dtype=np.float64)
    a, b = r6[..., :3], r6[..., 3:6]
    c1 = a / np.linalg.norm(a, axis=-1, keepdims=True)
    c2 = b - np.sum(c1 * b, axis=-1, keepdims=True) * c1
    c2 = c2 / np.linalg.norm(c2, axis=-1, keepdims=True)
    return np.stack([c1, c2, np.cross(c1, c2)], axis=-1)


def matrix_to_rotation6d(R) -> np.ndarray:
    R = np.asarray(R, dtype=np.float64)
    return np.concatenate([R[..., :, 0], R[..., :, 1]], axis=-1)


@dataclass
class CameraIntrinsics:
    """Pinhole, single shared focal."""
    focal: float
    cx: float
    cy: float
    width: int
    height: int

    def scaled(self, level: int) -> "CameraIntrinsics":
        s = 0.5 ** level
        return CameraIntrinsics(self.focal * s, (self.cx + 0.5) * s - 0.5, (self.cy + 0.5) * s - 0.5,
                                self.width >> level, self.height >> level)


@dataclass
class Pose:
    """x_cam = R x_world + t, rotation stored in the 6D representation."""
    rotation6d: np.ndarray
    translation: np.ndarray

    def __post_init__(self):
        self.rotation6d = np.asarray(self.rotation6d, dtype=np.float64).reshape(6)
        self.translation = np.asarray(self.translation, dtype=np.float64).reshape(3)

    @staticmethod
    def identity() -> "Pose":
        return Pose(np.array([1.0, 0.0, 0.0, 0.0, 1.0, 0.0]), np.zeros(3))

    @staticmethod
    def from_matrix(R, t) -> "Pose":
        return Pose(matrix_to_rotation6d(R), np.asarray(t, dtype=np.float64))

    @property
    def R(self) -> np.ndarray:
        return rotation6d_to_matrix(self.rotation6d)

    def compose(self, other: "Pose") -> "Pose":
        Ra = self.R
        return Pose.from_matrix(Ra @ other.R, Ra @ other.translation + self.translation)

    def inverse(self) -> "Pose":
        Rt = self.R.T
        return Pose.from_matrix(Rt, -Rt @ self.translation)

    def camera_center(self) -> np.ndarray:
        return -self.R.T @ self.translation

    def transform(self, pts) -> np.ndarray:
        return np.asarray(pts, dtype=np.float64) @ self.R.T + self.translation

    def copy(self) -> "Pose":
        return Pose(self.rotation6d.copy(), self.translation.copy())


def project(intr: CameraIntrinsics, pose: Pose, points):
    """World points (N,3) -> pixels (N,2) (NaN behind the camera), valid mask."""
    cam = pose.transform(np.atleast_2d(np.asarray(points, dtype=np.float64)))
    depth = cam[:, 2]
    valid = depth > 1e-12
    d = np.where(valid, depth, 1.0)
    px = np.stack([intr.focal * cam[:, 0] / d + intr.cx, intr.focal * cam[:, 1] / d + intr.cy], axis=1)
    px[~valid] = np.nan
    return px, valid


def unproject(intr: CameraIntrinsics, pose: Pose, pixels, depths) -> np.ndarray:
    px = np.atleast_2d(np.asarray(pixels, dtype=np.float64))
    d = np.asarray(depths, dtype=np.float64).reshape(-1)
    cam = np.stack([(px[:, 0] - intr.cx) / intr.focal * d, (px[:, 1] - intr.cy) / intr.focal * d, d],
                   axis=-1)
    return (cam - pose.translation) @ pose.R


def umeyama(src, dst, with_scale: bool = True):
    """Similarity (s, R, t) minimising ||dst - (s R src + t)||^2."""
    src = np.asarray(src, dtype=np.float64)
    dst = np.asarray(dst, dtype=np.float64)
    ms, md = src.mean(axis=0), dst.mean(axis=0)
    a, b = src - ms, dst - md
    Sigma = b.T @ a / len(src)
    U, D, Vt = np.linalg.svd(Sigma)
    E = np.ones(3)
    if np.linalg.det(U) * np.linalg.det(Vt) < 0:
        E[2] = -1.0
    R = (U * E) @ Vt
    s = 1.0
    if with_scale:
        var = float((a * a).sum()) / len(src)
        s = float((D * E).sum() / var) if var > 0 else 1.0
    return s, R, md - s * R @ ms


@dataclass
class Track:
    point: np.ndarray | None
    obs: list


class TrackTable:
    """Tracks with a per-track observation cap (the supervision window); the
    container bootstrap returns (reference scene.py:306-344)."""

    def __init__(self, n_obs_max: int = 6):
        self.n_obs_max = n_obs_max
        self.tracks: dict = {}
        self._by_obs: dict = {}
        self._next = 0

    def __len__(self) -> int:
        return len(self.tracks)

    def new_track(self, obs: list, point=None) -> int:
        if len(obs) < 2:
            raise ValueError("a track needs at least two observations")
        tid = self._next
        self._next += 1
        kept = list(obs)[-self.n_obs_max:]
        self.tracks[tid] = Track(point=point, obs=kept)
        for fr, kp, _, _ in kept:
            self._by_obs[(fr, kp)] = tid
        return tid

    def track_of(self, frame_index: int, kp_index: int):
        return self._by_obs.get((frame_index, kp_index))

    def add_observation(self, tid: int, frame_index: int, kp_index: int, x: float, y: float) -> None:
        tr = self.tracks[tid]
        tr.obs.append((frame_index, kp_index, x, y))
        while len(tr.obs) > self.n_obs_max:
            fr, kp, _, _ = tr.obs.pop(0)
            self._by_obs.pop((fr, kp), None)
        self._by_obs[(frame_index, kp_index)] = tid
