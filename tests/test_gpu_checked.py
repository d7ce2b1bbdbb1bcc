"""The checked build (libhgs_gpu_checked.so: HGS_DCHECK device bounds asserts
on every staged / scattered / gathered index of the hot kernels against the
capacities of the render's buffers) over every kernel family -- the
substitute for compute-sanitizer, which the GPU pool does not allow.  A
failed assert traps the kernel, so the run exits non-zero."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2505_13215_b200", "libhgs_gpu_checked.so")


@pytest.mark.gpu
@pytest.mark.parametrize("scale", [1, 4])
def test_checked_build_runs_every_kernel_family(scale):
    assert os.path.exists(LIB), "make -C paper_2505_13215_b200/csrc CHECKED=1"
    env = dict(os.environ, HGS_LIB=LIB, HGS_RUN_SCALE=str(scale))
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_run.py")], env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and "sanitize run ok" in r.stdout, (r.stdout[-2000:], r.stderr[-4000:])
    assert "HGS_CHECKED" not in r.stdout + r.stderr


def test_checked_library_is_built_with_the_asserts():
    """The checked library exists (built by __graft_entry__.build) and carries the assert strings."""
    assert os.path.exists(LIB)
    blob = open(LIB, "rb").read()
    assert b"HGS_CHECKED" in blob
