"""GPU parity of the blocked sweep in the Level-3 block orderings (reading R2-5 of
PAPER.md:1815-1824, Sec 6.4: the blocking principle "applied recursively further";
csrc/ordering.h) against the oracle's or_hz_blocked_ord with the same partition and
ordering, and the multi-rank schedule in them (loopback transport: block columns move only
between outer steps) bitwise equal to one rank."""
import numpy as np
import pytest

import oracle
from hostfactors import device_layout
from paper_1907_08560_b200 import inputs
from test_gpu_multirank_loopback import assert_same

pytestmark = pytest.mark.gpu

ORD = {"level3": oracle.ORDER_LEVEL3, "hier": oracle.ORDER_HIER}


@pytest.fixture(scope="module")
def gh():
    from paper_1907_08560_b200 import build, ghsvd
    build.build()
    return ghsvd


def relerr(a, b):
    a, b = np.sort(np.asarray(a)), np.sort(np.asarray(b))
    return float(np.max(np.abs(a - b) / np.abs(b)))


def residual(F, J, G, lam, Z):
    nf2 = np.linalg.norm(F) ** 2 + np.linalg.norm(G) ** 2
    Hx = F.conj().T @ (J[:, None] * (F @ Z))
    Sx = G.conj().T @ (G @ Z)
    return float((np.linalg.norm(Hx - Sx * lam[None, :], axis=0) / (nf2 * np.linalg.norm(Z, axis=0))).max())


def solve(gh, P, nblocks, ordering, nsup, variant="bo", want_x=False, **kw):
    m, n = P.F.shape
    c = gh.Context(m, n, variant=variant, nblocks=nblocks, ordering=ordering, super_blocks=nsup, max_sweeps=64,
                   want_x=want_x, **kw)
    c.set_factors(P.F, P.J, P.G)
    st = c.sweep()
    out = c.extract()
    X = c.extract_x() if want_x else None
    c.close()
    return st, out, X


@pytest.mark.parametrize("ordering,nblocks,nsup,variant", [("level3", 8, 4, "bo"), ("hier", 8, 4, "bo"),
                                                           ("level3", 16, 4, "bo"), ("hier", 16, 8, "bo"),
                                                           ("level3", 12, 6, "bo"), ("level3", 8, 4, "fb")])
def test_level3_orderings_match_oracle(gh, ordering, nblocks, nsup, variant):
    P = inputs.known_hyperbolic(14, 96, 64, 0.4)
    st, (lam, sf, sg, Z), _ = solve(gh, P, nblocks, ordering, nsup, variant)
    F0, J0, G0 = device_layout(P.F, P.J, P.G)
    Fo, Go, Zp, sto = oracle.hz_blocked(F0, J0, G0, nblocks, inner_sweeps=1 if variant == "bo" else 30,
                                        cmax=64, ordering=ORD[ordering], nsup=nsup)
    lo, *_ = oracle.extract(Fo, J0, Go, Zp)
    assert st["converged"] and sto["converged"]
    assert abs(st["sweeps"] - sto["sweeps"]) <= 1
    assert relerr(lam, lo) <= 1e-9
    assert relerr(lam, P.lam_true) <= 1e-9
    assert residual(P.F, P.J, P.G, lam, Z) <= 1e-12 * 64


@pytest.mark.parametrize("ordering,nsup", [("level3", 4), ("hier", 4)])
def test_level3_block_steps_elementwise(gh, ordering, nsup):
    """The first 10 block steps (across an outer-step boundary) elementwise against the
    oracle's block pivots (or_block_pair, Sec 6.4.2-6.4.3) applied in the oracle's ordering."""
    P = inputs.known_hyperbolic(31, 300, 128, 0.5)
    m, n = P.F.shape
    nblk, ns = 16, 10
    c = gh.Context(m, n, variant="bo", nblocks=nblk, ordering=ordering, super_blocks=nsup)
    c.set_factors(P.F, P.J, P.G)
    c.run_steps(0, ns)
    Fg, Gg, Zg = c.transformed(m, n)
    c.close()
    F, J0, G = device_layout(P.F, P.J, P.G)
    Z = np.asfortranarray(np.eye(n, dtype=complex))
    start, width = oracle.block_partition(n, nblk)
    for s in range(ns):
        for k in range(nblk // 2):
            p, q = oracle.order_pair(ORD[ordering], nblk, nsup, s, k)
            oracle.block_pair(F, J0, G, Z, start[p], width[p], start[q], width[q])
    for X, Y in ((Fg, F), (Gg, G), (Zg, Z)):
        assert (np.linalg.norm(X - Y, axis=0) / np.linalg.norm(Y, axis=0)).max() < 1e-10


@pytest.mark.parametrize("ordering,variant,want_x", [("hier", "bo", False), ("hier", "fb", False),
                                                    ("hier", "bo", True), ("level3", "bo", True)])
def test_level3_orderings_odd_n_fb_and_x(gh, ordering, variant, want_x):
    """Odd n (bordered to even order, Sec 6.3.2), FB inner sweeps, and X = Z^{-1} (NEXT-1)
    in the Level-3 orderings against the oracle's blocked sweep in the same ordering."""
    P = inputs.known_hyperbolic(35, 150, 63, 0.4)
    st, (lam, sf, sg, Z), X = solve(gh, P, 8, ordering, 4, variant, want_x=want_x)
    F0, J0, G0 = device_layout(P.F, P.J, P.G)
    Fo, Go, Zp, sto = oracle.hz_blocked(F0, J0, G0, 8, inner_sweeps=1 if variant == "bo" else 30, cmax=64,
                                        ordering=ORD[ordering], nsup=4)
    assert st["converged"] and sto["converged"] and abs(st["sweeps"] - sto["sweeps"]) <= 1
    assert relerr(lam, P.lam_true) <= 1e-9
    assert residual(P.F, P.J, P.G, lam, Z) <= 1e-12 * 63
    if want_x:
        assert np.abs(X @ Z - np.eye(63)).max() < 1e-10


def test_level3_round_robin_limits_bitwise(gh):
    """LEVEL3 with 2 super blocks (or one block column per super block), HIER with one block
    column per super block: the round-robin, bitwise."""
    P = inputs.known_hyperbolic(32, 200, 96, 0.4)
    ref = solve(gh, P, 8, "rr", 0)
    for ordering, nsup in (("level3", 2), ("level3", 8), ("hier", 8)):
        assert_same(solve(gh, P, 8, ordering, nsup), ref)


@pytest.mark.parametrize("ordering,world,nblocks", [("level3", 2, 16), ("hier", 2, 16), ("level3", 4, 16),
                                                    ("hier", 4, 32), ("level3", 2, 12)])
def test_level3_loopback_bitwise_equal_single(gh, ordering, world, nblocks):
    """One super pair per rank (super_blocks = 2 world): no exchange inside an outer step."""
    from test_gpu_multirank_loopback import multi
    P = inputs.known_hyperbolic(21, 400, 256, 0.4)
    nsup = 2 * world
    ref = solve(gh, P, nblocks, ordering, nsup)
    res = multi(gh, P, nblocks, world, False, f"l3{ordering}{world}_{nblocks}", ordering=ordering,
                super_blocks=nsup)
    for r in range(world):
        assert_same(res[r], ref)
    assert relerr(ref[1][0], P.lam_true) <= 1e-9


def test_level3_loopback_want_x_and_fewer_super_blocks(gh):
    """W travels with the outer-step exchanges; super_blocks = 4 on 4 ranks (a super pair
    split over two ranks: exchanges inside outer steps too) stays bitwise equal."""
    from test_gpu_multirank_loopback import multi
    P = inputs.known_hyperbolic(22, 300, 192, 0.5)
    ref = solve(gh, P, 16, "level3", 4, want_x=True)
    for world in (2, 4):
        res = multi(gh, P, 16, world, True, f"l3x{world}", ordering="level3", super_blocks=4)
        for r in range(world):
            assert_same(res[r], ref)


def test_level3_invalid_options(gh):
    P = inputs.known_hyperbolic(33, 96, 64, 0.4)
    with pytest.raises(gh.GHSVDError):
        gh.Context(96, 64, variant="pointwise", ordering="level3")
    with pytest.raises(gh.GHSVDError):
        solve(gh, P, 16, "level3", 6)     # 6 does not divide 16
    with pytest.raises(gh.GHSVDError):
        solve(gh, P, 24, "hier", 8)       # 3 block columns per super block
