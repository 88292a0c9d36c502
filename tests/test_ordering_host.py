"""Host logic of the Level-3 block orderings in libghsvd (csrc/ordering.h, comm.cpp; reading
R2-5 of PAPER.md:1815-1824, Sec 6.4) against the oracle's independent implementation
(oracle.order_pair, pinned by tests/test_oracle_ordering.py), and the exchange plans they
give.  No GPU needed: these entry points are host-only."""
import pytest

import oracle
from paper_1907_08560_b200 import ghsvd

CASES = [(4, 2), (8, 2), (8, 4), (8, 8), (16, 4), (16, 8), (24, 4), (32, 8), (64, 4), (64, 16), (128, 4),
         (128, 16), (12, 6)]


@pytest.mark.parametrize("ordering", ["rr", "level3", "hier"])
@pytest.mark.parametrize("nblk,nsup", CASES)
def test_product_ordering_equals_oracle(ordering, nblk, nsup):
    o = ghsvd.ORDERINGS[ordering]
    B = nblk // nsup
    if ordering == "hier" and B != 1 and B % 2:
        assert ghsvd.order_steps(ordering, nblk, nsup) == -1
        return
    nst = ghsvd.order_steps(ordering, nblk, nsup)
    assert nst == oracle.order_steps(o, nblk, nsup)
    for s in range(nst):
        for k in range(nblk // 2):
            assert ghsvd.order_pair(ordering, nblk, nsup, s, k) == oracle.order_pair(o, nblk, nsup, s, k)


def test_ordering_bad_arguments():
    assert ghsvd.order_steps("level3", 8, 3) == -1
    assert ghsvd.order_steps("level3", 8, 16) == -1
    assert ghsvd.order_steps("hier", 24, 8) == -1
    assert ghsvd.order_steps(5, 8, 4) == -1
    with pytest.raises(ghsvd.GHSVDError):
        ghsvd.order_pair("level3", 8, 4, ghsvd.order_steps("level3", 8, 4), 0)
    assert ghsvd.block_owner_ord("level3", 8, 4, 3, 0, 0) == -1   # world must divide nblk / 2


@pytest.mark.parametrize("ordering", ["level3", "hier"])
@pytest.mark.parametrize("nblk,world", [(8, 2), (16, 2), (32, 4), (64, 8), (128, 8)])
def test_level3_exchanges_only_between_outer_steps(ordering, nblk, world):
    """One super pair per rank (super_blocks = 2 world): the exchange plans are empty inside
    an outer step; 2 world - 1 exchanges per sweep (the round-robin: nblk - 1).  Every plan
    is consistent: what rank r sends to r' is what r' receives from r."""
    nsup = 2 * world
    nst = ghsvd.order_steps(ordering, nblk, nsup)
    moving = 0
    for s in range(nst):
        sn = (s + 1) % nst
        plans = [ghsvd.exchange_plan(nblk, world, r, s, sn, ordering, nsup) for r in range(world)]
        sent = sorted((b, r, p) for r, (snd, _) in enumerate(plans) for b, p in snd)
        recv = sorted((b, p, r) for r, (_, rcv) in enumerate(plans) for b, p in rcv)
        assert sent == recv
        moving += bool(sent)
        for b in range(nblk):   # owners agree with the plans
            o1 = ghsvd.block_owner_ord(ordering, nblk, nsup, world, s, b)
            o2 = ghsvd.block_owner_ord(ordering, nblk, nsup, world, sn, b)
            assert (o1 != o2) == any(x[0] == b for x in sent)
    assert moving == 2 * world - 1
    rr_moving = sum(1 for s in range(nblk - 1)
                    if any(ghsvd.exchange_plan(nblk, world, r, s, (s + 1) % (nblk - 1))[0] for r in range(world)))
    assert rr_moving == nblk - 1
