"""One context, several problems (the serving pattern): after a solve, set_factors with a
new (possibly smaller, odd-n) problem within the context's capacity must give bitwise the
result of a fresh context -- no state (Z', counters, block partition, graph cache, bordering
column, Phase-2 permutation) leaks from one problem into the next."""
import numpy as np
import pytest

from paper_1907_08560_b200 import inputs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gh():
    from paper_1907_08560_b200 import build, ghsvd
    build.build()
    return ghsvd


def solve(ctx, P):
    ctx.set_factors(P.F, P.J, P.G)
    st = ctx.sweep()
    lam, sf, sg, Z = ctx.extract()
    return st, lam, Z


@pytest.mark.parametrize("variant", ["pointwise", "bo"])
def test_context_reuse_bitwise_equal_fresh(gh, variant):
    probs = [inputs.known_hyperbolic(31, 400, 256, 0.4), inputs.known_hyperbolic(32, 300, 191, 0.5),
             inputs.random_pencil(33, 384, 256, 0.5), inputs.known_gsvd(34, 200, 128)]
    shared = gh.Context(400, 256, variant=variant, max_sweeps=40)
    for P in probs:
        m, n = P.F.shape
        st_a, lam_a, Z_a = solve(shared, P)
        fresh = gh.Context(m, n, variant=variant, max_sweeps=40)
        st_b, lam_b, Z_b = solve(fresh, P)
        fresh.close()
        assert st_a["sweeps"] == st_b["sweeps"] and st_a["converged"]
        assert st_a["transforms_all"] == st_b["transforms_all"]
        np.testing.assert_array_equal(lam_a, lam_b)
        np.testing.assert_array_equal(Z_a, Z_b)
    shared.close()


def test_context_reuse_after_reduce(gh):
    """A Phase-2 problem (P2 permutation, m -> n) followed by a direct problem."""
    kind, at = inputs.make_config(0)
    NA, NL, NG = at.A.shape
    ctx = gh.Context(2 * NA * NL, NG, NL, variant="pointwise")
    ctx.factor(at.A, at.B, at.U, at.TAA, at.TAB, at.TBB)
    ctx.reduce()
    ctx.sweep()
    P = inputs.known_gsvd(35, 16, 12)
    st_a, lam_a, Z_a = solve(ctx, P)
    fresh = gh.Context(16, 12, variant="pointwise")
    st_b, lam_b, Z_b = solve(fresh, P)
    np.testing.assert_array_equal(lam_a, lam_b)
    np.testing.assert_array_equal(Z_a, Z_b)
    ctx.close()
    fresh.close()
