"""GPU parity of ghsvd_factor (Phase 1, Algorithm 1) against the oracle's or_factor."""
import numpy as np
import pytest

import oracle
from paper_1907_08560_b200 import inputs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gh():
    from paper_1907_08560_b200 import build, ghsvd
    build.build()
    return ghsvd


def _sorted_rows(F, J):
    order = np.concatenate([np.where(J > 0)[0], np.where(J < 0)[0]])
    return F[order], J[order]


@pytest.mark.parametrize("NA,NL,NG,neg", [(2, 4, 12, 0.5), (3, 5, 20, 0.4), (16, 49, 96, 39 / 98), (5, 81, 64, 0.5),
                                          (2, 121, 40, 0.5)])
def test_factor_matches_oracle(gh, NA, NL, NG, neg):
    at = inputs.lapw_atoms(70 + NL, NA, NL, NG, neg)
    Fo, Jo, Go = oracle.factor(at.A, at.B, at.U, at.TAA, at.TAB, at.TBB)
    Fo_s, Jo_s = _sorted_rows(Fo, Jo)
    m = 2 * NA * NL
    ctx = gh.Context(m, NG, NL)
    ctx.factor(at.A, at.B, at.U, at.TAA, at.TAB, at.TBB)
    F, J, G, p2 = ctx.get_factors()
    if NG % 2:
        F, G, J = F[:-1, :-1], G[:-1, :-1], J[:-1]
    assert np.array_equal(J, Jo_s)
    assert np.array_equal(G, Go)                       # [A_a; U_a B_a] exactly
    assert np.abs(F - Fo_s).max() <= 1e-12 * np.abs(Fo).max()
    ctx.close()


def test_config0_end_to_end(gh):
    """BASELINE configs[0] through the C ABI: factor -> sweep -> extract vs the oracle pipeline."""
    kind, at = inputs.make_config(0)
    ctx = gh.Context(16, 12, 4)
    ctx.factor(at.A, at.B, at.U, at.TAA, at.TAB, at.TBB)
    st = ctx.sweep()
    lam, sf, sg, Z = ctx.extract()
    F0, J0, G0 = oracle.factor(at.A, at.B, at.U, at.TAA, at.TAB, at.TBB)   # the oracle's own Phase 1
    Fo, Go, Zp, sto = oracle.hz_pointwise(F0, J0, G0)
    lo, *_ = oracle.extract(Fo, J0, Go, Zp)
    assert st["converged"] and abs(st["sweeps"] - sto["sweeps"]) <= 1
    assert np.max(np.abs(np.sort(lam) - np.sort(lo)) / np.abs(np.sort(lo))) <= 1e-9
    ctx.close()


def test_singular_T_rejected(gh):
    at = inputs.lapw_atoms(3, 2, 3, 6, 0.5)
    at.TAA[1][:] = 0
    at.TAB[1][:] = 0
    at.TBB[1][:] = 0
    ctx = gh.Context(12, 6, 3)
    with pytest.raises(gh.GHSVDError) as e:
        ctx.factor(at.A, at.B, at.U, at.TAA, at.TAB, at.TBB)
    assert e.value.status == -7
    ctx.close()
