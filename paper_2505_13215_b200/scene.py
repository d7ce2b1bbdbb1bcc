"""Host-side scene and camera containers (mirror of the reference's value types).

The reference stores a scene as two ``std::vector``s of AoS double structs
(``Gaussian4D``/``Gaussian3D`` in include/hgs/scene.hpp:13-59, with a heap
``std::vector<Vec3>`` of SH coefficients each, sh.hpp:15-22) and the camera as
a pinhole struct (include/hgs/camera.hpp:11-31).  This module keeps the same
fields and meaning but as one numpy array per parameter class ("host SoA"),
which is the layout the C-ABI ``hgs_scene_upload`` consumes and the one the
oracle's ctypes wrapper consumes, so both sides of every parity test see the
same numbers.

Shapes (K = (sh_degree+1)**2):
  dynamics: mean_x (n4,3), mean_t (n4,), ql (n4,4), qr (n4,4) (w,x,y,z),
            log_s4 (n4,4) = (s_x,s_y,s_z,s_t), op4 (n4,) opacity logit,
            sh4 (n4,K,3)
  statics:  mean3 (n3,3), quat3 (n3,4), log_s3 (n3,3), op3 (n3,), sh3 (n3,K,3)
"""
from __future__ import annotations

import copy
import math
from dataclasses import dataclass, field

import numpy as np

SH_C0 = 0.28209479177387814  # sh.cpp:10


def sh_coeff_count(degree: int) -> int:
    """sh.hpp:12"""
    return (degree + 1) * (degree + 1)


@dataclass
class HybridScene:
    """HybridScene (scene.hpp:49-59) as per-class numpy arrays."""

    sh_degree: int = 1
    tau: float = 0.5
    duration_seconds: float = 1.0
    extent: float = 1.0
    mean_x: np.ndarray = field(default_factory=lambda: np.zeros((0, 3)))
    mean_t: np.ndarray = field(default_factory=lambda: np.zeros((0,)))
    ql: np.ndarray = field(default_factory=lambda: np.zeros((0, 4)))
    qr: np.ndarray = field(default_factory=lambda: np.zeros((0, 4)))
    log_s4: np.ndarray = field(default_factory=lambda: np.zeros((0, 4)))
    op4: np.ndarray = field(default_factory=lambda: np.zeros((0,)))
    sh4: np.ndarray | None = None
    mean3: np.ndarray = field(default_factory=lambda: np.zeros((0, 3)))
    quat3: np.ndarray = field(default_factory=lambda: np.zeros((0, 4)))
    log_s3: np.ndarray = field(default_factory=lambda: np.zeros((0, 3)))
    op3: np.ndarray = field(default_factory=lambda: np.zeros((0,)))
    sh3: np.ndarray | None = None

    DYN_FIELDS = ("mean_x", "mean_t", "ql", "qr", "log_s4", "op4", "sh4")
    STA_FIELDS = ("mean3", "quat3", "log_s3", "op3", "sh3")

    def __post_init__(self):
        K = sh_coeff_count(self.sh_degree)
        if self.sh4 is None:
            self.sh4 = np.zeros((len(self.mean_t), K, 3))
        if self.sh3 is None:
            self.sh3 = np.zeros((len(self.op3), K, 3))
        for f in self.DYN_FIELDS + self.STA_FIELDS:
            setattr(self, f, np.ascontiguousarray(getattr(self, f), dtype=np.float64))

    @property
    def n4(self) -> int:
        return int(self.mean_t.shape[0])

    @property
    def n3(self) -> int:
        return int(self.op3.shape[0])

    def total(self) -> int:  # scene.hpp:58
        return self.n3 + self.n4

    def copy(self) -> "HybridScene":
        return copy.deepcopy(self)

    def subset(self, n4: int, n3: int) -> "HybridScene":
        """The first n4 dynamic and n3 static Gaussians (a bounded sample)."""
        out = self.copy()
        for f in self.DYN_FIELDS:
            setattr(out, f, np.ascontiguousarray(getattr(self, f)[:n4]))
        for f in self.STA_FIELDS:
            setattr(out, f, np.ascontiguousarray(getattr(self, f)[:n3]))
        return out

    def as_float32_exact(self) -> "HybridScene":
        """Round every parameter to float32 and widen back.

        The device stores parameters in FP32 (SoA); feeding the FP64 oracle the
        widened values makes both sides consume bit-identical inputs.
        """
        out = self.copy()
        for f in self.DYN_FIELDS + self.STA_FIELDS:
            setattr(out, f, getattr(out, f).astype(np.float32).astype(np.float64))
        return out

    def validate_shapes(self) -> None:
        K = sh_coeff_count(self.sh_degree)
        n4, n3 = self.n4, self.n3
        exp = dict(mean_x=(n4, 3), mean_t=(n4,), ql=(n4, 4), qr=(n4, 4), log_s4=(n4, 4),
                   op4=(n4,), sh4=(n4, K, 3), mean3=(n3, 3), quat3=(n3, 4), log_s3=(n3, 3),
                   op3=(n3,), sh3=(n3, K, 3))
        for k, shp in exp.items():
            got = getattr(self, k).shape
            if got != shp:
                raise ValueError(f"HybridScene.{k}: shape {got}, expected {shp}")


@dataclass
class Camera:
    """Pinhole camera, x_cam = R x + t (camera.hpp:11-31)."""

    fx: float = 0.0
    fy: float = 0.0
    cx: float = 0.0
    cy: float = 0.0
    rot: np.ndarray = field(default_factory=lambda: np.eye(3))
    trans: np.ndarray = field(default_factory=lambda: np.zeros(3))
    width: int = 0
    height: int = 0
    near: float = 0.01
    far: float = 100.0

    def position(self) -> np.ndarray:  # camera.hpp:19
        return -self.rot.T @ self.trans

    def validate(self) -> None:  # camera.hpp:21-26
        if not (self.fx > 0.0 and self.fy > 0.0):
            raise ValueError("Camera: fx, fy must be positive")
        if not (0.0 < self.near < self.far):
            raise ValueError("Camera: need 0 < near < far")
        if self.width <= 0 or self.height <= 0:
            raise ValueError("Camera: bad image dimensions")
        r = np.asarray(self.rot, dtype=np.float64)
        if (np.abs(r.T @ r - np.eye(3)).max() > 1e-8 or abs(np.linalg.det(r) - 1.0) > 1e-8):
            raise ValueError("Camera: rotation not orthonormal")

    @staticmethod
    def look_at(eye, target, up, focal: float, width: int, height: int) -> "Camera":
        """camera.cpp:6-22 (same operation order, scalar by scalar)."""
        eye = [float(v) for v in eye]
        target = [float(v) for v in target]
        up = [float(v) for v in up]

        def normalized(v):
            n = math.sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2])
            return [v[0] / n, v[1] / n, v[2] / n]

        def cross(a, b):
            return [a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0]]

        fwd = normalized([target[i] - eye[i] for i in range(3)])
        right = normalized(cross(fwd, up))
        down = cross(fwd, right)
        rot = np.array([right, down, fwd], dtype=np.float64)
        trans = np.zeros(3)
        for i in range(3):
            s = (-rot[i, 0]) * eye[0]
            s = s + (-rot[i, 1]) * eye[1]
            s = s + (-rot[i, 2]) * eye[2]
            trans[i] = s
        return Camera(fx=float(focal), fy=float(focal), cx=width / 2.0, cy=height / 2.0,
                      rot=rot, trans=trans, width=int(width), height=int(height))


# ---------------------------------------------------------------------------
# Synthetic inputs of the BASELINE.json configs.
# ---------------------------------------------------------------------------

def _unit_quats(rng: np.random.Generator, n: int) -> np.ndarray:
    q = rng.standard_normal((n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    q[q[:, 0] < 0] *= -1.0  # canonical sign (gauss_math.cpp:13-24)
    return q


def synthetic_scene(n4: int, n3: int, sh_degree: int = 3, seed: int = 0,
                    density_n: int | None = None, tau: float = 0.5) -> HybridScene:
    """random_scene distributions (tests/oracles.hpp:63-97), density-scaled.

    means ~ N(0, 1.2^2); quats normalised N(0,1)^4; opacity = logit(U(0.05,0.95));
    mu_t ~ U(0,1); exp(s_t) ~ U(0.08, 0.58); SH DC from rgb ~ U(0,1), higher
    bands 0.2 N(0,1); spatial scales exp(s) ~ U(0.05,0.35) * (100/N)^(1/3)
    (SURVEY.md 8d).  Values are rounded to float32 (the device precision).
    """
    rng = np.random.default_rng(seed)
    N = density_n if density_n is not None else max(n4 + n3, 1)
    shrink = (100.0 / N) ** (1.0 / 3.0)
    K = sh_coeff_count(sh_degree)

    def sh_block(n):
        sh = np.zeros((n, K, 3))
        sh[:, 0, :] = (rng.uniform(0.0, 1.0, (n, 3)) - 0.5) / SH_C0
        if K > 1:
            sh[:, 1:, :] = 0.2 * rng.standard_normal((n, K - 1, 3))
        return sh

    def logit(p):
        return np.log(p / (1.0 - p))

    s = HybridScene(sh_degree=sh_degree, tau=tau, extent=2.0)
    s.mean_x = 1.2 * rng.standard_normal((n4, 3))
    s.mean_t = rng.uniform(0.0, 1.0, n4)
    s.ql = _unit_quats(rng, n4)
    s.qr = _unit_quats(rng, n4)
    ls = np.log(rng.uniform(0.05, 0.35, (n4, 3)) * shrink)
    lt = np.log(rng.uniform(0.08, 0.58, (n4, 1)))
    s.log_s4 = np.concatenate([ls, lt], axis=1)
    s.op4 = logit(rng.uniform(0.05, 0.95, n4))
    s.sh4 = sh_block(n4)
    s.mean3 = 1.2 * rng.standard_normal((n3, 3))
    s.quat3 = _unit_quats(rng, n3)
    s.log_s3 = np.log(rng.uniform(0.05, 0.35, (n3, 3)) * shrink)
    s.op3 = logit(rng.uniform(0.05, 0.95, n3))
    s.sh3 = sh_block(n3)
    s.__post_init__()
    return s.as_float32_exact()


def ring_camera(seed: int, width: int, height: int, index: int | None = None,
                n_ring: int = 16) -> Camera:
    """random_camera (tests/oracles.hpp:99-108) with focal = 60*W/64.

    With ``index`` set, the azimuth is the index-th of ``n_ring`` evenly spaced
    ring positions (the c4 16-camera ring).
    """
    rng = np.random.default_rng(seed + 7919)
    a = 2.0 * math.pi * rng.uniform()
    h = -1.5 + 3.0 * rng.uniform()
    r = 4.0 + 2.0 * rng.uniform()
    if index is not None:
        a = 2.0 * math.pi * index / n_ring
    eye = (r * math.cos(a), h, r * math.sin(a))
    return Camera.look_at(eye, (0.0, 0.0, 0.0), (0.0, -1.0, 0.0), 60.0 * width / 64.0,
                          width, height)


# The five BASELINE.json configurations (SURVEY.md 8d "Per-config inputs").
CONFIGS = {
    "c1": dict(n4=100_000, n3=0, width=640, height=480, seed=1, t=0.5),
    "c2": dict(n4=240_000, n3=60_000, width=1352, height=1014, seed=2, t=0.5),
    "c3": dict(n4=300_000, n3=0, width=1352, height=1014, seed=3, t=0.5),
    "c4": dict(n4=1_600_000, n3=400_000, width=1352, height=1014, seed=4, t=0.5),
    "c5": dict(n4=3_200_000, n3=800_000, width=2048, height=1088, seed=5, t=0.5),
}
