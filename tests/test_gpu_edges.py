"""Degenerate and boundary inputs through the C ABI (both variants): a single column
(n = 1, bordered to a single pivot pair, C-10), empty and over-capacity inputs (rejected),
J = +I and J = -I (definite H of either sign), and a zero column of F (pointwise: lambda = 0,
H may be singular, only S must be definite; blocked: the singular block
pivot stops the process)."""
import numpy as np
import pytest

import oracle
from hostfactors import device_layout
from paper_1907_08560_b200 import inputs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gh():
    from paper_1907_08560_b200 import build, ghsvd
    build.build()
    return ghsvd


def relerr(a, b):
    a, b = np.sort(np.asarray(a)), np.sort(np.asarray(b))
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300)))


@pytest.mark.parametrize("variant", ["pointwise", "bo"])
def test_single_column(gh, variant):
    rng = np.random.default_rng(5)
    m = 9
    F = (rng.standard_normal((m, 1)) + 1j * rng.standard_normal((m, 1))) / np.sqrt(2)
    G = (rng.standard_normal((m, 1)) + 1j * rng.standard_normal((m, 1))) / np.sqrt(2)
    J = np.where(rng.random(m) < 0.5, -1, 1).astype(np.int8)
    ctx = gh.Context(m, 1, variant=variant)
    ctx.set_factors(F, J, G)
    st = ctx.sweep()
    lam, sf, sg, Z = ctx.extract()
    ctx.close()
    h = float(np.real(np.vdot(F[:, 0], J * F[:, 0])))
    s = float(np.real(np.vdot(G[:, 0], G[:, 0])))
    assert st["converged"] and lam.shape == (1,) and Z.shape == (1, 1)
    assert abs(lam[0] - h / s) <= 1e-14 * abs(h / s)
    # Z = 1 / Sigma with Sigma = sqrt(|h| + s) (eq 3.2 for one column)
    assert abs(abs(Z[0, 0]) - 1.0 / np.sqrt(abs(h) + s)) <= 1e-14 / np.sqrt(abs(h) + s)


@pytest.mark.parametrize("m,n", [(0, 0), (4, 0), (0, 4), (3, 4)])
def test_empty_and_wide_inputs_rejected(gh, m, n):
    ctx = gh.Context(8, 4)
    F = np.zeros((m, n), np.complex128)
    with pytest.raises(gh.GHSVDError) as e:
        ctx.set_factors(F, np.ones(m, np.int8), F)
    assert e.value.status == -1
    ctx.close()


def test_over_capacity_rejected_and_capacity_accepted(gh):
    ctx = gh.Context(40, 16, variant="bo")
    P = inputs.random_pencil(6, 41, 16, 0.5)
    with pytest.raises(gh.GHSVDError) as e:
        ctx.set_factors(P.F, P.J, P.G)
    assert e.value.status == -1
    P = inputs.random_pencil(6, 40, 17, 0.5)
    with pytest.raises(gh.GHSVDError):
        ctx.set_factors(P.F, P.J, P.G)
    P = inputs.random_pencil(6, 40, 16, 0.5)
    ctx.set_factors(P.F, P.J, P.G)
    assert ctx.sweep()["converged"]
    ctx.close()


@pytest.mark.parametrize("variant", ["pointwise", "bo"])
@pytest.mark.parametrize("sign", [1, -1])
def test_definite_H_of_either_sign(gh, variant, sign):
    P = inputs.random_pencil(9, 120, 64, 0.0)
    J = np.full(120, sign, np.int8)
    ctx = gh.Context(120, 64, variant=variant)
    ctx.set_factors(P.F, J, P.G)
    F0, J0, G0 = device_layout(P.F, J, P.G)
    st = ctx.sweep()
    lam, *_ = ctx.extract()
    ctx.close()
    Fo, Go, Zp, _ = oracle.hz_pointwise(F0, J0, G0)
    lo, *_ = oracle.extract(Fo, J0, Go, Zp)
    assert st["converged"] and np.all(np.sign(lam) == sign)
    assert relerr(lam, lo) <= 1e-9


def test_zero_column_of_F_blocked_stops_rank_deficient(gh):
    """Blocked: the block pivot H_blk = F_pair^* J F_pair is singular, and "the
    factorization should reveal if H is rank deficient, in which case the process stops"
     -- GHSVD_E_RANK_DEFICIENT, not a silent result."""
    P = inputs.random_pencil(10, 100, 48, 0.5)
    F = P.F.copy()
    F[:, 7] = 0.0
    ctx = gh.Context(100, 48, variant="bo")
    ctx.set_factors(F, P.J, P.G)
    with pytest.raises(gh.GHSVDError) as e:
        ctx.sweep()
    assert e.value.status == -7
    ctx.close()


@pytest.mark.parametrize("variant", ["pointwise"])
def test_zero_column_of_F_gives_zero_eigenvalue(gh, variant):
    P = inputs.random_pencil(10, 100, 48, 0.5)
    F = P.F.copy()
    F[:, 7] = 0.0
    ctx = gh.Context(100, 48, variant=variant)
    ctx.set_factors(F, P.J, P.G)
    F0, J0, G0 = device_layout(F, P.J, P.G)
    st = ctx.sweep()
    lam, *_ = ctx.extract()
    ctx.close()
    Fo, Go, Zp, _ = oracle.hz_pointwise(F0, J0, G0)
    lo, *_ = oracle.extract(Fo, J0, Go, Zp)
    assert st["converged"]
    k = int(np.argmin(np.abs(lam)))
    assert abs(lam[k]) <= 1e-12 * np.abs(lam).max()
    nz = np.abs(lo) > 1e-12 * np.abs(lo).max()
    a, b = np.sort(lam[np.abs(lam) > 1e-12 * np.abs(lam).max()]), np.sort(lo[nz])
    assert a.shape == b.shape and relerr(a, b) <= 1e-9


def test_reduce_all_nan_F_reports_nonfinite(gh):
    """Phase 2's JQR pivot search with every J-norm NaN: GHSVD_E_NONFINITE, no fault
    (the argmax sentinel used to index a column)."""
    P = inputs.random_pencil(12, 60, 16, 0.5)
    F = np.full_like(P.F, np.nan)
    ctx = gh.Context(60, 16)
    ctx.set_factors(F, P.J, P.G)
    with pytest.raises(gh.GHSVDError) as e:
        ctx.reduce()
    assert e.value.status == -8
    ctx.close()
    # the device is still usable afterwards
    ctx = gh.Context(60, 16)
    ctx.set_factors(P.F, P.J, P.G)
    ctx.reduce()
    assert ctx.sweep()["converged"]
    ctx.close()
