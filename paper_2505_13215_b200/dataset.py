"""Dataset ingest: the on-disk multi-view format of
data_io.cpp:44-177 and the binary PPM frames of image.cpp:35-75.

Layout (docs/formats.md of the reference): root/cameras.txt (one camera per
line: id fx fy cx cy width height near far, 9 rotation entries row-major, 3
translation entries), optional root/meta.txt (key = value: duration_seconds,
background_r/g/b), optional root/points.txt (x y z r g b per line) and
root/camXX/frame_%05d.ppm.

B200-first difference: frames are kept as the 8-bit sRGB codes the files
hold (``frames="u8"``, the default) and decoded on the GPU inside the loss
(HGS_U8) -- 4x less host memory and host->device traffic than linear floats.
``frames="linear"`` returns read_ppm's float64 linear images instead (the
same values: srgb8_to_linear of the same bytes).  PPM decoding is native
(hgs_ppm_read_batch, a host thread pool writing straight into one
contiguous -- optionally pinned -- array per camera).
"""
from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass, field

import numpy as np

from . import _capi
from .scene import Camera
from .train import SRGB8_LUT, Frame, MultiViewDataset

__all__ = ["FormatError", "KeyValueFile", "InitPoints", "ppm_info", "read_ppm_u8", "read_ppm", "write_ppm",
           "read_ppm_batch", "load_points", "save_points", "load_dataset", "save_dataset"]

FormatError = _capi.FormatError


def _check(rc: int) -> None:
    if rc != 0:
        raise _capi._STATUS.get(rc, _capi.HgsError)(_capi.lib().hgs_image_last_error().decode())


# ---------------------------------------------------------------- PPM frames
def ppm_info(path: str) -> tuple[int, int]:
    """(width, height) of a P6 file (read_ppm's header rules)."""
    w, h = C.c_int32(), C.c_int32()
    _check(_capi.lib().hgs_ppm_info(os.fsencode(path), C.byref(w), C.byref(h)))
    return w.value, h.value


def read_ppm_u8(path: str) -> np.ndarray:
    """The (h, w, 3) uint8 sRGB codes of a P6 file."""
    w, h = ppm_info(path)
    out = np.empty((h, w, 3), dtype=np.uint8)
    _check(_capi.lib().hgs_ppm_read(os.fsencode(path), out.ctypes.data_as(C.POINTER(C.c_uint8)), w, h))
    return out


def read_ppm(path: str) -> np.ndarray:
    """read_ppm (image.cpp:49-75): (h, w, 3) float64 linear RGB."""
    return SRGB8_LUT[read_ppm_u8(path)]


def write_ppm(img: np.ndarray, path: str) -> None:
    """write_ppm (image.cpp:35-47): linear float images are quantised with
    linear_to_srgb8; uint8 arrays are written as sRGB codes."""
    a = np.ascontiguousarray(img)
    if a.ndim != 3 or a.shape[2] != 3:
        raise ValueError("write_ppm: expected an (h, w, 3) image")
    if a.dtype == np.uint8:
        code = _capi.HGS_U8
    elif a.dtype == np.float32:
        code = _capi.HGS_F32
    else:
        a = a.astype(np.float64, copy=False)
        code = _capi.HGS_F64
    _check(_capi.lib().hgs_ppm_write(os.fsencode(path), a.ctypes.data_as(C.c_void_p), code, a.shape[1], a.shape[0]))


def read_ppm_batch(paths: list[str], width: int, height: int, out: np.ndarray | None = None,
                   threads: int = 0) -> np.ndarray:
    """Reads n frames of one size into ``out`` ((n, h, w, 3) uint8; e.g. a
    pinned buffer's numpy view) on ``threads`` host threads (0 = all)."""
    n = len(paths)
    if out is None:
        out = np.empty((n, height, width, 3), dtype=np.uint8)
    if out.shape != (n, height, width, 3) or out.dtype != np.uint8 or not out.flags.c_contiguous:
        raise ValueError("read_ppm_batch: out must be a contiguous (n, h, w, 3) uint8 array")
    enc = [os.fsencode(p) for p in paths]
    parr = (C.c_char_p * max(1, n))(*enc)
    stride = height * width * 3
    base = out.ctypes.data
    oarr = (C.POINTER(C.c_uint8) * max(1, n))(*[C.cast(C.c_void_p(base + i * stride), C.POINTER(C.c_uint8))
                                                 for i in range(n)])
    _check(_capi.lib().hgs_ppm_read_batch(parr, n, oarr, width, height, threads))
    return out


# ----------------------------------------------------------- key = value files
class KeyValueFile:
    """config.cpp:22-110: '#' comments, key = value lines, duplicate keys and
    (at finish) unused keys are FormatErrors."""

    def __init__(self, path: str):
        self.path = path
        self.values: dict[str, str] = {}
        self.used: dict[str, bool] = {}
        try:
            f = open(path)
        except OSError as e:
            raise FormatError(f"config: cannot open {path}") from e
        with f:
            for lineno, line in enumerate(f, 1):
                line = line.rstrip("\n")
                if "#" in line:
                    line = line[: line.index("#")]
                line = line.strip()
                if not line:
                    continue
                if "=" not in line:
                    raise FormatError(f"{path}:{lineno}: expected key=value")
                key, val = line.split("=", 1)
                key, val = key.strip(), val.strip()
                if not key or not val:
                    raise FormatError(f"{path}:{lineno}: empty key or value")
                if key in self.values:
                    raise FormatError(f"{path}:{lineno}: duplicate key {key}")
                self.values[key] = val
                self.used[key] = False

    def _find(self, key: str):
        if key not in self.values:
            return None
        self.used[key] = True
        return self.values[key]

    def get_float(self, key: str, default: float) -> float:
        v = self._find(key)
        if v is None:
            return default
        if v == "inf":
            return math.inf
        try:
            return float(v)
        except ValueError:
            raise FormatError(f"{self.path}: key {key}: not a number: {v}") from None

    def get_int(self, key: str, default: int) -> int:
        v = self._find(key)
        if v is None:
            return default
        try:
            return int(v)
        except ValueError:
            raise FormatError(f"{self.path}: key {key}: not an integer: {v}") from None

    def get_bool(self, key: str, default: bool) -> bool:
        v = self._find(key)
        if v is None:
            return default
        if v in ("true", "1"):
            return True
        if v in ("false", "0"):
            return False
        raise FormatError(f"{self.path}: key {key}: expected true/false: {v}")

    def get_uint(self, key: str, default: int) -> int:
        v = self._find(key)
        if v is None:
            return default
        try:
            x = int(v)
            if x < 0 or x >= 1 << 64:
                raise ValueError
            return x
        except ValueError:
            raise FormatError(f"{self.path}: key {key}: not an unsigned integer: {v}") from None

    def finish(self) -> None:
        unknown = [k for k in sorted(self.used) if not self.used[k]]
        if unknown:
            raise FormatError(f"{self.path}: unknown keys: " + ", ".join(unknown))


# -------------------------------------------------------------------- points
@dataclass
class InitPoints:  # data_io.hpp InitPoint list, as arrays
    positions: np.ndarray = field(default_factory=lambda: np.zeros((0, 3)))
    rgb: np.ndarray = field(default_factory=lambda: np.zeros((0, 3)))

    def __len__(self) -> int:
        return int(self.positions.shape[0])


def load_points(path: str) -> InitPoints:
    """load_points (data_io.cpp:160-177)"""
    try:
        f = open(path)
    except OSError as e:
        raise FormatError(f"load_points: cannot open {path}") from e
    pos, rgb = [], []
    with f:
        for lineno, line in enumerate(f, 1):
            line = line.rstrip("\n")
            if not line or line[0] == "#":
                continue
            tok = line.split()
            try:
                v = [float(t) for t in tok[:6]]
                if len(v) != 6:
                    raise ValueError
            except ValueError:
                raise FormatError(f"{path}:{lineno}: expected x y z r g b") from None
            pos.append(v[:3])
            rgb.append(v[3:])
    return InitPoints(np.array(pos, dtype=np.float64).reshape(-1, 3), np.array(rgb, dtype=np.float64).reshape(-1, 3))


def save_points(points: InitPoints, path: str) -> None:
    """save_points (data_io.cpp:179-187), 17 significant digits"""
    with open(path, "w") as f:
        for p, c in zip(points.positions, points.rgb):
            f.write(" ".join(f"{float(v):.17g}" for v in (*p, *c)) + "\n")


# ------------------------------------------------------------------ datasets
def _cam_dir(cid: int) -> str:
    return f"cam{cid:02d}"


def _frame_name(j: int) -> str:
    return f"frame_{j:05d}.ppm"


def _frame_time(j: int, n: int) -> float:  # data_io.cpp:37-39
    return j / (n - 1) if n > 1 else 0.0


def save_dataset(ds: MultiViewDataset, root: str) -> None:
    """save_dataset (data_io.cpp:44-76)"""
    os.makedirs(root, exist_ok=True)
    ids = ds.camera_ids or list(range(len(ds.cameras)))
    with open(os.path.join(root, "cameras.txt"), "w") as f:
        for cid, c in zip(ids, ds.cameras):
            r = np.asarray(c.rot, dtype=np.float64).reshape(9)
            t = np.asarray(c.trans, dtype=np.float64).reshape(3)
            nums = [c.fx, c.fy, c.cx, c.cy]
            f.write(f"{cid} " + " ".join(f"{float(v):.17g}" for v in nums) + f" {c.width} {c.height} " +
                    " ".join(f"{float(v):.17g}" for v in [c.near, c.far, *r, *t]) + "\n")
    with open(os.path.join(root, "meta.txt"), "w") as f:
        f.write(f"duration_seconds = {float(ds.duration_seconds):.17g}\n")
        for k, v in zip("rgb", ds.background):
            f.write(f"background_{k} = {float(v):.17g}\n")
    for cid, frames in zip(ids, ds.frames):
        d = os.path.join(root, _cam_dir(cid))
        os.makedirs(d, exist_ok=True)
        for j, fr in enumerate(frames):
            write_ppm(fr.image, os.path.join(d, _frame_name(j)))
    if ds.init_points is not None and len(ds.init_points):
        save_points(ds.init_points, os.path.join(root, "points.txt"))


def _parse_cameras(root: str) -> tuple[list[Camera], list[int]]:
    path = os.path.join(root, "cameras.txt")
    try:
        f = open(path)
    except OSError as e:
        raise FormatError(f"load_dataset: cannot open {path}") from e
    cams, ids = [], []
    with f:
        for lineno, line in enumerate(f, 1):
            line = line.rstrip("\n")
            if not line or line[0] == "#":
                continue
            tok = line.split()
            try:
                if len(tok) < 21:  # the id and 20 numbers
                    raise ValueError
                cid = int(tok[0])
                fx, fy, cx, cy = (float(t) for t in tok[1:5])
                w, h = int(tok[5]), int(tok[6])
                near, far = float(tok[7]), float(tok[8])
                rot = np.array([float(t) for t in tok[9:18]]).reshape(3, 3)
                trans = np.array([float(t) for t in tok[18:21]])
            except ValueError:
                raise FormatError(f"{path}:{lineno}: expected 21 numbers after the camera id") from None
            c = Camera(fx=fx, fy=fy, cx=cx, cy=cy, rot=rot, trans=trans, width=w, height=h, near=near, far=far)
            try:
                c.validate()
            except ValueError as e:
                raise FormatError(f"{path}:{lineno}: {e}") from None
            cams.append(c)
            ids.append(cid)
    if not cams:
        raise FormatError(f"{path}: no cameras")
    return cams, ids


def load_dataset(root: str, held_out_camera: int = -1, frames: str = "u8", pinned: bool = False,
                 threads: int = 0) -> tuple[MultiViewDataset, MultiViewDataset]:
    """load_dataset (data_io.cpp:78-158) -> (train split, held-out split).

    frames: "u8" keeps the sRGB codes (train on the device with HGS_U8),
    "linear" decodes to float64 like read_ppm.  pinned: frame arrays live in
    page-locked host memory (torch) for asynchronous host->device copies."""
    if frames not in ("u8", "linear"):
        raise ValueError("load_dataset: frames is 'u8' or 'linear'")
    cams, ids = _parse_cameras(root)
    meta = os.path.join(root, "meta.txt")
    duration, bg = 1.0, [0.0, 0.0, 0.0]
    if os.path.exists(meta):
        kv = KeyValueFile(meta)
        duration = kv.get_float("duration_seconds", duration)
        bg = [kv.get_float(f"background_{k}", v) for k, v in zip("rgb", bg)]
        kv.finish()
    pts_path = os.path.join(root, "points.txt")
    points = load_points(pts_path) if os.path.exists(pts_path) else InitPoints()

    all_frames = []
    expected = None
    for cam, cid in zip(cams, ids):
        d = os.path.join(root, _cam_dir(cid))
        paths = []
        while os.path.exists(os.path.join(d, _frame_name(len(paths)))):
            paths.append(os.path.join(d, _frame_name(len(paths))))
        if not paths:
            raise FormatError(f"{d}: no frames found")
        for p in paths:  # header check first: the reference's error for a size mismatch
            if ppm_info(p) != (cam.width, cam.height):
                raise FormatError(f"{p}: frame size disagrees with cameras.txt")
        if expected is None:
            expected = len(paths)
        if len(paths) != expected:
            raise FormatError(f"{d}: frame count differs between cameras")
        shape = (len(paths), cam.height, cam.width, 3)
        if pinned:
            import torch

            buf = torch.empty(shape, dtype=torch.uint8).pin_memory().numpy()
        else:
            buf = np.empty(shape, dtype=np.uint8)
        read_ppm_batch(paths, cam.width, cam.height, out=buf, threads=threads)
        imgs = buf if frames == "u8" else SRGB8_LUT[buf]
        all_frames.append([Frame(time=_frame_time(j, expected), image=imgs[j]) for j in range(len(paths))])

    train = MultiViewDataset(cameras=[], frames=[], background=tuple(bg), duration_seconds=duration,
                             camera_ids=[], init_points=points)
    held = MultiViewDataset(cameras=[], frames=[], background=tuple(bg), duration_seconds=duration,
                            camera_ids=[], init_points=InitPoints())
    found = False
    for cam, cid, fr in zip(cams, ids, all_frames):
        dst = held if cid == held_out_camera else train
        found |= cid == held_out_camera
        dst.cameras.append(cam)
        dst.camera_ids.append(cid)
        dst.frames.append(fr)
    if held_out_camera >= 0 and not found:
        raise FormatError(f"load_dataset: held-out camera id {held_out_camera} not in dataset")
    if not train.cameras:
        raise FormatError("load_dataset: holding out the only camera leaves nothing to train on")
    return train, held
