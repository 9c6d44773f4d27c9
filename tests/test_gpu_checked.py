"""Every kernel (ingest, k_heavy, k_tiles, k_fix, readout, PageRank, Power-NF, unpermute; the
serial and the overlapped plan) run by
the device bounds-checked build (lib/libpsi_checked.so, -DPSI_CHECKS: label, row, slot, panel
and leader indices are checked and trap on a violation) -- the stand-in for compute-sanitizer,
which is closed on the GPU pool."""

import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

pytestmark = pytest.mark.gpu


def test_checked_build_runs_every_kernel(gpu):
    from paper_2206_09960_b200 import _build
    _build.build(checked=True)
    env = dict(os.environ, PSI_LIB="checked")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_small.py")],
                         capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-2000:]
    assert "PSI_CHECKS" not in out.stdout + out.stderr
    assert out.stdout.count("sum(psi)=") == 4 and "overlapped=1" in out.stdout
