"""Pins of the oracle's block orderings (reading R2-5: the Level-2 blocking principle of
PAPER.md:1815-1824, Sec 6.4, "applied recursively further") and of the blocked sweep run in
them.  The orderings are checked by brute force against their definitions (every step a
perfect matching of the block columns, the multiplicity of every block pair per sweep,
super-pair locality) and against the round-robin they reduce to; the sweeps against
spectra known by construction (inputs.known_hyperbolic / known_gsvd)."""
import itertools

import numpy as np
import pytest

import oracle
from paper_1907_08560_b200 import inputs

L3, HIER, RR = oracle.ORDER_LEVEL3, oracle.ORDER_HIER, oracle.ORDER_RR


def relerr(a, b):
    a = np.sort(np.asarray(a))
    b = np.sort(np.asarray(b))
    return float(np.max(np.abs(a - b) / np.abs(b)))


def steps(ordering, nblk, nsup):
    nst = oracle.order_steps(ordering, nblk, nsup)
    return [[oracle.order_pair(ordering, nblk, nsup, s, k) for k in range(nblk // 2)] for s in range(nst)]


CASES = [(4, 2), (8, 2), (8, 4), (8, 8), (16, 4), (16, 8), (24, 4), (32, 8), (32, 16), (64, 4), (12, 6)]


@pytest.mark.parametrize("ordering", [L3, HIER])
@pytest.mark.parametrize("nblk,nsup", CASES)
def test_ordering_steps_are_perfect_matchings(ordering, nblk, nsup):
    B = nblk // nsup
    if ordering == HIER and B != 1 and B % 2:
        with pytest.raises(oracle.OracleError):
            oracle.order_steps(ordering, nblk, nsup)
        return
    S = steps(ordering, nblk, nsup)
    Q = nsup // 2
    want = (2 * Q - 1) * (2 * B - 1) if ordering == L3 else (B - 1) + (2 * Q - 1) * B
    assert len(S) == want
    for st in S:
        blocks = [b for pq in st for b in pq]
        assert sorted(blocks) == list(range(nblk))   # disjoint pairs covering every block
        assert all(p < q for p, q in st)


@pytest.mark.parametrize("nblk,nsup", CASES)
def test_pair_multiplicity_per_sweep(nblk, nsup):
    """HIER: every block pair exactly once per sweep (as the round-robin).  LEVEL3: pairs of
    one super block once per outer step (2Q - 1 times), pairs across super blocks once."""
    B, Q = nblk // nsup, nsup // 2
    for ordering in (L3, HIER):
        if ordering == HIER and B != 1 and B % 2:
            continue
        cnt = {}
        for st in steps(ordering, nblk, nsup):
            for pq in st:
                cnt[pq] = cnt.get(pq, 0) + 1
        for p, q in itertools.combinations(range(nblk), 2):
            same = p // B == q // B
            want = (2 * Q - 1 if same else 1) if ordering == L3 else 1
            assert cnt.get((p, q), 0) == want, (ordering, p, q)


@pytest.mark.parametrize("ordering", [L3, HIER])
@pytest.mark.parametrize("nblk,nsup", [(8, 4), (16, 4), (16, 8), (32, 8), (64, 4)])
def test_super_pair_locality(ordering, nblk, nsup):
    """Slots [u B, (u+1) B) hold the block columns of one super pair, fixed for the whole
    outer step: with P = Q ranks owning one super pair each, block columns change owner
    only between outer steps (2Q - 1 times per sweep, counting the wrap to the next
    sweep), instead of after every one of the nblk - 1 round-robin steps."""
    B, Q = nblk // nsup, nsup // 2
    if ordering == HIER and B != 1 and B % 2:
        return
    S = steps(ordering, nblk, nsup)
    owned = [[frozenset(b for pq in st[u * B:(u + 1) * B] for b in pq) for u in range(Q)] for st in S]
    for own in owned:
        for u in range(Q):
            assert len(own[u]) == 2 * B
            P_, Q_ = sorted({b // B for b in own[u]})   # two whole super blocks
            assert own[u] == frozenset(range(P_ * B, P_ * B + B)) | frozenset(range(Q_ * B, Q_ * B + B))
    changes = sum(owned[s] != owned[(s + 1) % len(S)] for s in range(len(S)))
    assert changes == (2 * Q - 1 if Q > 1 else 0)
    rr_changes = sum(1 for s in range(nblk - 1)
                     if {oracle.rr_pair(nblk, s, k) for k in range(nblk // 2)} !=
                     {oracle.rr_pair(nblk, (s + 1) % (nblk - 1), k) for k in range(nblk // 2)})
    assert rr_changes == nblk - 1 or nblk == 2


@pytest.mark.parametrize("nblk", [4, 8, 16, 32])
def test_orderings_reduce_to_round_robin(nblk):
    """LEVEL3 with nsup = 2 (one super pair) or nsup = nblk (super blocks of one block
    column), and HIER with nsup = nblk, are the Level-2 round-robin (C-11)."""
    rr = [[oracle.rr_pair(nblk, s, k) for k in range(nblk // 2)] for s in range(nblk - 1)]
    assert steps(L3, nblk, 2) == rr
    assert steps(L3, nblk, nblk) == rr
    assert steps(HIER, nblk, nblk) == rr
    assert steps(RR, nblk, 0) == rr


def test_ordering_argument_errors():
    for args in [(L3, 8, 3), (L3, 8, 0), (L3, 8, 16), (HIER, 24, 8), (7, 8, 4), (L3, 7, 2)]:
        with pytest.raises(oracle.OracleError):
            oracle.order_steps(*args)
    with pytest.raises(oracle.OracleError):
        oracle.order_pair(L3, 8, 4, oracle.order_steps(L3, 8, 4), 0)


@pytest.mark.parametrize("ordering,nblk,nsup,inner", [(L3, 8, 4, 1), (HIER, 8, 4, 1), (L3, 16, 4, 1),
                                                     (HIER, 16, 8, 1), (L3, 12, 6, 1), (L3, 8, 4, 30)])
def test_blocked_sweep_in_level3_orderings_known_spectrum(ordering, nblk, nsup, inner):
    """The blocked BO / FB sweep in the Level-3 orderings converges to the spectrum known
    by construction (J != I, and J = I), with the same stop rule (C-3)."""
    P = inputs.known_hyperbolic(14, 96, 64, 0.4)
    F, G, Zp, st = oracle.hz_blocked(P.F, P.J, P.G, nblk, inner_sweeps=inner, ordering=ordering, nsup=nsup)
    lam, *_ = oracle.extract(F, P.J, G, Zp)
    assert st["converged"] and st["big_per_sweep"][st["sweeps"] - 1] == 0
    assert relerr(lam, P.lam_true) < 1e-10
    assert np.linalg.norm(F - P.F @ Zp) / np.linalg.norm(F) < 1e-11   # a congruence
    Q = inputs.known_gsvd(15, 80, 48)
    F, G, Zp, st = oracle.hz_blocked(Q.F, Q.J, Q.G, 8, ordering=ordering, nsup=4)
    lam, *_ = oracle.extract(F, Q.J, G, Zp)
    assert st["converged"] and relerr(lam, Q.lam_true) < 1e-10


def test_blocked_round_robin_via_ordering_entry_is_bitwise_level2():
    P = inputs.known_hyperbolic(16, 64, 48, 0.5)
    a = oracle.hz_blocked(P.F, P.J, P.G, 6)
    b = oracle.hz_blocked(P.F, P.J, P.G, 6, ordering=L3, nsup=2)   # reduces to round-robin
    for x, y in zip(a[:3], b[:3]):
        assert np.array_equal(x, y)
    assert a[3]["sweeps"] == b[3]["sweeps"]
