"""The C ABI used from plain C (examples/c_demo.c, no Python in the process): random
complex J-GHSVD problems through the pointwise and the blocked BO sweep, every eigenpair's
residual <= 1e-12 n checked in C from the inputs (BASELINE north_star bound)."""
import subprocess

import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("m,n", [(320, 192), (517, 257)])
def test_c_demo_runs(m, n):
    from paper_1907_08560_b200 import build
    exe = build.build_c_demo()
    r = subprocess.run([exe, str(m), str(n)], capture_output=True, text=True, timeout=600)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count(" OK") == 2
