"""Writes the small golden fixtures of tests/golden/ (run once; committed).

  ckpt_small.hgsc     -- oracle.checkpoint.encode_checkpoint of a fixed
                         6-static / 5-dynamic degree-1 scene (oracle.Rng(7))
                         with a deterministic optimizer state: the byte layout
                         of data_io.cpp:444-719, frozen.
  ckpt_small.json     -- the values it holds (sha256 of the file + scalars).
  frame_5x3.ppm       -- a hand-written P6 frame with a header comment.

The fixtures pin the product's readers and writers against a frozen byte
stream independent of the code under test (tests/test_golden_cpu.py)."""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle as O  # noqa: E402
from oracle import checkpoint as CK  # noqa: E402
from paper_2505_13215_b200.scene import HybridScene  # noqa: E402


def golden_scene():
    s = O.Rng(7).random_scene(6, 5, 1)
    s.tau, s.duration_seconds, s.extent = 0.45, 1.75, 2.5
    return s


def golden_state(s):
    st = CK.State(s)
    k = 0
    for f in HybridScene.DYN_FIELDS + HybridScene.STA_FIELDS:
        a = getattr(st.m, f)
        a[...] = (np.arange(a.size).reshape(a.shape) + k) * 0.125
        getattr(st.v, f)[...] = np.abs(a) * 0.5 + 1.0
        k += 100
    st.grad_norm3 = np.arange(s.n3) * 0.25
    st.grad_norm4 = np.arange(s.n4) * 0.5
    st.count3 = np.arange(s.n3, dtype=np.uint32) * 3
    st.count4 = np.arange(s.n4, dtype=np.uint32) * 2
    st.step, st.skipped_nonfinite = 321, 4
    return st


if __name__ == "__main__":
    s = golden_scene()
    b = CK.encode_checkpoint(s, golden_state(s))
    open(os.path.join(HERE, "ckpt_small.hgsc"), "wb").write(b)
    json.dump({"sha256": hashlib.sha256(b).hexdigest(), "bytes": len(b), "n4": s.n4, "n3": s.n3, "sh_degree": 1,
               "tau": 0.45, "duration_seconds": 1.75, "extent": 2.5, "step": 321, "skipped_nonfinite": 4},
              open(os.path.join(HERE, "ckpt_small.json"), "w"), indent=1)
    pix = bytes([(7 * i + 3) % 256 for i in range(5 * 3 * 3)])
    open(os.path.join(HERE, "frame_5x3.ppm"), "wb").write(b"P6\n# golden\n5 3\n255\n" + pix)
    print("wrote", len(b), "bytes")
