"""The dense tensor-core group attend (attend_dense_tc_kernel, alaya_tc_attend.cuh)
against the CPU oracle on every small parity case: a subprocess runs the
parity and fuzz suites with the group candidate format forced on
(ALAYA_GFMT=1, so beta = 110 and below take the dense path too), covering
ragged prefixes (partial last tiles), windows inside and outside the chunk,
GQA groups 1..8 and batches of sessions. The 128K beta = 140 cases of
test_gpu_parity_large.py run the same kernel by default."""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.parametrize("dense", ["1", "0"])
def test_group_format_paths_vs_oracle(cuda_ok, dense):
    env = dict(os.environ, ALAYA_GFMT="1", ALAYA_GRP_DENSE=dense)
    cmd = [sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider",
           "tests/test_gpu_parity.py", "tests/test_gpu_fuzz.py"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " passed" in r.stdout and "failed" not in r.stdout
