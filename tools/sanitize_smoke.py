"""Small run of every kernel family for compute-sanitizer (memcheck / racecheck / synccheck):
pointwise kernels 1-3 (cluster sizes 1 and 4, odd n bordered), blocked BO and FB, Phase 1,
Phase 2, extraction, the 2x2 batch hook.  Exits non-zero on any wrong result."""
import os
import sys
import warnings

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1907_08560_b200 import build, ghsvd, inputs  # noqa: E402

warnings.simplefilter("ignore")
build.build()


def check(lam, ref, tol=1e-8):
    e = np.max(np.abs(np.sort(lam) - np.sort(ref)) / np.abs(np.sort(ref)))
    assert e < tol, e


P = inputs.known_hyperbolic(3, 130, 61, 0.4)      # odd n -> bordering
for kernel, cluster in ((1, 1), (2, 1), (3, 1), (1, 4), (2, 4), (3, 4)):
    ctx = ghsvd.Context(130, 61, kernel=kernel, cluster=cluster)
    ctx.set_factors(P.F, P.J, P.G)
    ctx.sweep()
    lam, *_ = ctx.extract()
    ctx.close()
    check(lam, P.lam_true)
for variant, nb in (("bo", 4), ("fb", 6)):
    ctx = ghsvd.Context(130, 61, variant=variant, nblocks=nb)
    ctx.set_factors(P.F, P.J, P.G)
    ctx.sweep()
    lam, *_ = ctx.extract()
    ctx.close()
    check(lam, P.lam_true)
for env in ({"GHSVD_PIVOT_CL": "1"}, {"GHSVD_GROUPS": "2"}, {"GHSVD_GRAM3M": "0"}, {"GHSVD_SERIAL": "1"}):
    os.environ.update(env)
    ctx = ghsvd.Context(130, 61, variant="bo", nblocks=6, want_x=True)
    ctx.set_factors(P.F, P.J, P.G)
    ctx.sweep()
    lam, *_ = ctx.extract()
    X = ctx.extract_x()
    ctx.close()
    check(lam, P.lam_true)
    for k in env:
        del os.environ[k]
at = inputs.lapw_atoms(5, 3, 6, 20, 0.5)
ctx = ghsvd.Context(36, 20, 6, variant="bo", nblocks=2)
ctx.factor(at.A, at.B, at.U, at.TAA, at.TAB, at.TBB)
ctx.reduce(colpiv=True)
ctx.sweep()
lam, *_ = ctx.extract()
ctx.close()
ctx = ghsvd.Context(36, 20, 6, variant="bo", nblocks=2)
ctx.factor(at.A, at.B, at.U, at.TAA, at.TAB, at.TBB)
ctx.reduce()
ctx.sweep()
lam, *_ = ctx.extract()
ctx.close()
ctx = ghsvd.Context(16, 8)
z, k = ctx.hz2x2_batch(np.array([[1, 2, 0.3, 0.1, 1, 1, 0.2, 0.0]] * 64), 1e-15)
ctx.close()
print("sanitize smoke OK")
