"""Restatement of the reference's .hgsc checkpoint format -- TEST INFRASTRUCTURE ONLY.

Follows data_io.cpp:444-719 (ByteWriter/ByteReader, encode_scene /
decode_scene, encode_state / decode_state, save_checkpoint /
load_checkpoint) with struct + zlib.crc32 (the reference links zlib's crc32,
data_io.cpp:4, 650-652).  Byte layout, all little-endian:

    "HGSC" u32 version(=1)
    section*: tag[4] u64 len u32 crc32(payload) payload[len]
    SCEN: u32 deg f64 tau f64 duration f64 extent u64 n3 u64 n4
          statics  : 3 mean, 4 quat (w,x,y,z), 3 log_scales, 1 opacity, u32 deg, 3K sh
          dynamics : 3 mean_x, 1 mean_t, 4 ql, 4 qr, 4 log_scales, 1 opacity, u32 deg, 3K sh
    OPTS: u64 step u64 skipped, 12 x (f64v m, f64v v) in the order
          statics mean quat scales opacity sh, dynamics mean_x mean_t
          quat_left quat_right scales opacity sh; f64v grad_norm3, grad_norm4;
          u32v count3, count4        (f64v/u32v = u64 length + data)

Only tests/ use this module; the product implements the format natively
(paper_2505_13215_b200/csrc/checkpoint.cu).
"""
from __future__ import annotations

import math
import struct
import zlib

import numpy as np

from paper_2505_13215_b200.scene import HybridScene, sh_coeff_count

VERSION = 1  # data_io.cpp:448
MAX_SH_DEGREE = 3


class FormatError(RuntimeError):
    pass


class IntegrityError(RuntimeError):
    pass


class UnsupportedVersionError(RuntimeError):
    pass


STA_CLASSES = (("mean3", 3), ("quat3", 4), ("log_s3", 3), ("op3", 1), ("sh3", -1))
DYN_CLASSES = (("mean_x", 3), ("mean_t", 1), ("ql", 4), ("qr", 4), ("log_s4", 4), ("op4", 1), ("sh4", -1))


def _rows(scene: HybridScene, name: str, dim: int) -> np.ndarray:
    K3 = 3 * sh_coeff_count(scene.sh_degree)
    a = np.asarray(getattr(scene, name), dtype=np.float64)
    n = scene.n3 if name in dict(STA_CLASSES) else scene.n4
    return a.reshape(n, K3 if dim < 0 else dim)


def encode_scene(scene: HybridScene) -> bytes:
    """data_io.cpp:527-551"""
    out = [struct.pack("<Idddqq", scene.sh_degree, scene.tau, scene.duration_seconds, scene.extent,
                       scene.n3, scene.n4)]
    deg = struct.pack("<I", scene.sh_degree)
    for classes, n in ((STA_CLASSES, scene.n3), (DYN_CLASSES, scene.n4)):
        parts = [_rows(scene, name, dim) for name, dim in classes]
        head = np.concatenate(parts[:-1], axis=1)  # every f64 field before the SH degree
        for i in range(n):
            out.append(head[i].astype("<f8").tobytes())
            out.append(deg)
            out.append(parts[-1][i].astype("<f8").tobytes())
    return b"".join(out)


def encode_state(scene: HybridScene, st) -> bytes:
    """data_io.cpp:597-619; ``st`` has m, v (scene-shaped), grad_norm3/4,
    count3/4, step, skipped_nonfinite (oracle.AdamState)."""
    out = [struct.pack("<QQ", st.step, st.skipped_nonfinite)]

    def f64v(a):
        a = np.ascontiguousarray(a, dtype="<f8").ravel()
        out.append(struct.pack("<Q", a.size))
        out.append(a.tobytes())

    def u32v(a):
        a = np.ascontiguousarray(a, dtype="<u4").ravel()
        out.append(struct.pack("<Q", a.size))
        out.append(a.tobytes())

    for name, dim in STA_CLASSES + DYN_CLASSES:
        f64v(_rows(st.m, name, dim))
        f64v(_rows(st.v, name, dim))
    f64v(st.grad_norm3)
    f64v(st.grad_norm4)
    u32v(st.count3)
    u32v(st.count4)
    return b"".join(out)


def _section(tag: bytes, payload: bytes) -> bytes:
    return tag + struct.pack("<QI", len(payload), zlib.crc32(payload) & 0xFFFFFFFF) + payload


def encode_checkpoint(scene: HybridScene, state=None) -> bytes:
    """save_checkpoint (data_io.cpp:656-665) as bytes."""
    b = b"HGSC" + struct.pack("<I", VERSION) + _section(b"SCEN", encode_scene(scene))
    if state is not None:
        b += _section(b"OPTS", encode_state(scene, state))
    return b


def save_checkpoint(scene: HybridScene, state, path: str) -> None:
    with open(path, "wb") as f:
        f.write(encode_checkpoint(scene, state))


class _Reader:  # data_io.cpp:466-494
    def __init__(self, buf: bytes):
        self.b, self.off = buf, 0

    def take(self, n: int) -> bytes:
        if self.off + n > len(self.b):
            raise FormatError("checkpoint: truncated section payload")
        v = self.b[self.off:self.off + n]
        self.off += n
        return v

    def u32(self):
        return struct.unpack("<I", self.take(4))[0]

    def u64(self):
        return struct.unpack("<Q", self.take(8))[0]

    def f64(self):
        return struct.unpack("<d", self.take(8))[0]

    def f64s(self, n):
        return np.frombuffer(self.take(8 * n), dtype="<f8").astype(np.float64)

    def f64v(self):
        n = self.u64()
        if n > len(self.b) // 8 + 1:
            raise FormatError("checkpoint: implausible array length")
        return self.f64s(n)

    def u32v(self):
        n = self.u64()
        if n > len(self.b) // 4 + 1:
            raise FormatError("checkpoint: implausible array length")
        return np.frombuffer(self.take(4 * n), dtype="<u4").astype(np.uint32)

    def done(self):
        return self.off == len(self.b)


def _get_quat(q: np.ndarray) -> np.ndarray:
    """data_io.cpp:500-511: validate without renormalising, flip to the
    canonical hemisphere (exact)."""
    w, x, y, z = (float(v) for v in q)
    n = math.sqrt(w * w + x * x + y * y + z * z)
    if not (abs(n - 1.0) <= 1e-6):
        raise FormatError("checkpoint: non-unit quaternion")
    flip = w < 0.0 or (w == 0.0 and (x < 0.0 or (x == 0.0 and (y < 0.0 or (y == 0.0 and z < 0.0)))))
    return -q if flip else q


def decode_scene(r: _Reader) -> HybridScene:
    """data_io.cpp:553-583 (a uniform SH degree per scene)"""
    deg = r.u32()
    if deg > MAX_SH_DEGREE:
        raise FormatError("checkpoint: bad scene SH degree")
    tau, duration, extent = r.f64(), r.f64(), r.f64()
    n3, n4 = r.u64(), r.u64()
    K = sh_coeff_count(deg)
    s = HybridScene(sh_degree=deg, tau=tau, duration_seconds=duration, extent=extent)
    for classes, n in ((STA_CLASSES, n3), (DYN_CLASSES, n4)):
        cols = {name: np.zeros((n, 3 * K if dim < 0 else dim)) for name, dim in classes}
        for i in range(n):
            for name, dim in classes:
                if dim < 0:
                    d = r.u32()
                    if d > MAX_SH_DEGREE:
                        raise FormatError("checkpoint: bad SH degree")
                    if d != deg:
                        raise FormatError("checkpoint: SH degree of a Gaussian differs from the scene's")
                    cols[name][i] = r.f64s(3 * K)
                else:
                    v = r.f64s(dim)
                    if name in ("quat3", "ql", "qr"):
                        v = _get_quat(v)
                    cols[name][i] = v
        for name, dim in classes:
            a = cols[name]
            if dim < 0:
                a = a.reshape(n, K, 3)
            elif dim == 1:
                a = a.reshape(n)
            setattr(s, name, a)
    if not r.done():
        raise FormatError("checkpoint: trailing bytes in scene section")
    return s


class State:
    """GradAccum as read back (m, v scene-shaped)."""

    def __init__(self, scene: HybridScene):
        self.m = _zeros_like(scene)
        self.v = _zeros_like(scene)
        self.grad_norm3 = np.zeros(scene.n3)
        self.grad_norm4 = np.zeros(scene.n4)
        self.count3 = np.zeros(scene.n3, np.uint32)
        self.count4 = np.zeros(scene.n4, np.uint32)
        self.step = 0
        self.skipped_nonfinite = 0


def _zeros_like(scene: HybridScene) -> HybridScene:
    s = scene.copy()
    for f in HybridScene.DYN_FIELDS + HybridScene.STA_FIELDS:
        getattr(s, f)[...] = 0.0
    return s


def decode_state(r: _Reader, scene: HybridScene) -> State:
    """data_io.cpp:621-643 + the consistency check of 711-717 (extended to
    every array: the device layout needs them all)."""
    st = State(scene)
    st.step, st.skipped_nonfinite = r.u64(), r.u64()
    K3 = 3 * sh_coeff_count(scene.sh_degree)
    for name, dim in STA_CLASSES + DYN_CLASSES:
        m, v = r.f64v(), r.f64v()
        if m.size != v.size:
            raise FormatError("checkpoint: moment size mismatch")
        n = scene.n3 if (name, dim) in STA_CLASSES else scene.n4
        d = K3 if dim < 0 else dim
        if m.size != n * d:
            raise FormatError("load_checkpoint: optimizer state disagrees with scene")
        shape = getattr(scene, name).shape
        getattr(st.m, name)[...] = m.reshape(shape)
        getattr(st.v, name)[...] = v.reshape(shape)
    st.grad_norm3, st.grad_norm4 = r.f64v(), r.f64v()
    st.count3, st.count4 = r.u32v(), r.u32v()
    if not r.done():
        raise FormatError("checkpoint: trailing bytes in state section")
    if st.grad_norm3.size != scene.n3 or st.grad_norm4.size != scene.n4 or st.count3.size != scene.n3 or \
            st.count4.size != scene.n4:
        raise FormatError("load_checkpoint: optimizer state disagrees with scene")
    return st


def decode_checkpoint(b: bytes):
    """load_checkpoint (data_io.cpp:667-719) over bytes -> (scene, state|None)."""
    if len(b) < 4 or b[:4] != b"HGSC":
        raise FormatError("load_checkpoint: bad magic")
    if len(b) < 8:
        raise FormatError("load_checkpoint: truncated header")
    version = struct.unpack("<I", b[4:8])[0]
    if version != VERSION:
        raise UnsupportedVersionError(f"load_checkpoint: unsupported version {version}")
    off = 8
    scene = None
    state_payload = None
    while off < len(b):
        if off + 16 > len(b):
            raise FormatError("load_checkpoint: truncated section header")
        tag = b[off:off + 4]
        ln, crc = struct.unpack("<QI", b[off + 4:off + 16])
        off += 16
        if off + ln > len(b):
            raise FormatError("load_checkpoint: truncated section payload")
        payload = b[off:off + ln]
        off += ln
        if zlib.crc32(payload) & 0xFFFFFFFF != crc:
            raise IntegrityError("load_checkpoint: checksum mismatch")
        if tag == b"SCEN":
            scene = decode_scene(_Reader(payload))
        elif tag == b"OPTS":
            state_payload = payload  # decoded against the scene below
    if scene is None:
        raise FormatError("load_checkpoint: no scene section")
    state = decode_state(_Reader(state_payload), scene) if state_payload is not None else None
    return scene, state


def load_checkpoint(path: str):
    try:
        with open(path, "rb") as f:
            b = f.read()
    except OSError as e:
        raise FormatError(f"load_checkpoint: cannot open {path}") from e
    return decode_checkpoint(b)
