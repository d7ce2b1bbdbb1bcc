"""gm::Rcp (K1's shared-reciprocal FP64 divisions) is bit-identical to IEEE
division: tools/div_exact.cu compares the two on random finite bit patterns
and on geometry-like magnitudes (every quotient, bit for bit)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_shared_reciprocal_division_is_bit_exact(tmp_path):
    exe = str(tmp_path / "div_exact")
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-fmad=false", "-o", exe,
                           os.path.join(ROOT, "tools", "div_exact.cu")], cwd=os.path.join(ROOT, "tools"))
    out = subprocess.run([exe, "8"], capture_output=True, text=True, timeout=300).stdout
    lines = [l for l in out.splitlines() if l.startswith("mode")]
    assert len(lines) == 2, out
    for l in lines:
        assert l.split(":")[1].strip().startswith("0 mismatches"), l
