"""Device fp64 helpers that re-implement IEEE operations must be bit-identical
to them: the shared-reciprocal V3 / double of dmath.cuh against three plain
divisions, over 2^28 random operand triples (all exponents, zeros, denormals,
infinities, NaNs).  Builds tests/cuda/div3_check.cu with nvcc and runs it."""
import os
import shutil
import subprocess

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.gpu
def test_v3_division_matches_ieee(tmp_path):
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    exe = tmp_path / "div3_check"
    subprocess.run([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "--fmad=false", "-o", str(exe),
                    os.path.join(HERE, "cuda", "div3_check.cu")], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and r.stdout.startswith("mismatches 0 "), r.stdout + r.stderr
