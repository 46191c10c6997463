"""The round-2 alternative layouts (csrc/Makefile ALTFLAGS: wide iterations of fp64 single-
source fields in the BFS-position layout, the change-driven worklist for every field kind),
built beside the product library as libgeodist_b200_alt.so: the GPU parity suite, run against
that build in a subprocess, must pass bit for bit as it does for the product build."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ALT = os.path.join(ROOT, "paper_1810_08218_b200", "libgeodist_b200_alt.so")


def test_alternative_layouts_parity_suite():
    assert os.path.exists(ALT), "libgeodist_b200_alt.so missing: __graft_entry__.build() makes it"
    env = dict(os.environ, GEODIST_B200_LIB=ALT)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                        os.path.join(ROOT, "tests", "test_gpu_parity.py")],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " passed" in r.stdout
