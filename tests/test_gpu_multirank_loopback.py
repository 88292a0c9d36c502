"""The multi-GPU blocked sweep (Sec 6.4.3) run on
ONE GPU through the loopback transport (include/ghsvd.h, nccl_id).

P contexts in this process, one host thread each, play the P ranks: each owns the
round-robin slots ghsvd_block_owner assigns to it, runs the multi-rank halves schedule on
its own stream, and after every block step pulls the block columns of F, G, Z (and W)
it receives from their previous owner (the ncclSend / ncclRecv pair's effect), with the
counters combined once per sweep and the outputs gathered at extraction.  No kernel waits
on another rank's kernel (CUDA events + a host barrier order the copies), so the ranks
may share the GPU.  Every block pair's arithmetic is the same in any launch grouping and
the Gram split is planned from the global pair count, so the result must be BITWISE equal
to the single-rank solve with the same partition -- a missing or stale block column, a
wrong owner or a wrong stop decision breaks equality.
"""
import threading

import numpy as np
import pytest

from paper_1907_08560_b200 import inputs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gh():
    from paper_1907_08560_b200 import build, ghsvd
    build.build()
    return ghsvd


def load(c, P):
    if hasattr(P, "F"):
        c.set_factors(P.F, P.J, P.G)
    else:   # Phase-1 atoms: every rank factors the same atoms (deterministic, no comm)
        c.factor(P.A, P.B, P.U, P.TAA, P.TAB, P.TBB)


def shape(P):
    if hasattr(P, "F"):
        return P.F.shape[0], P.F.shape[1], 0
    NA, NL, NG = P.A.shape
    return 2 * NA * NL, NG, NL


def single(gh, P, nblocks, want_x, variant="bo"):
    m, n, nl = shape(P)
    c = gh.Context(m, n, nl, variant=variant, nblocks=nblocks, max_sweeps=64, want_x=want_x)
    load(c, P)
    st = c.sweep()
    out = c.extract()
    X = c.extract_x() if want_x else None
    c.close()
    return st, out, X


def multi(gh, P, nblocks, world, want_x, key, variant="bo", local=False, **kw):
    import torch
    m, n, nl = shape(P)
    streams = [torch.cuda.Stream() for _ in range(world)]
    lid = gh.loopback_id(key)
    ctxs = [gh.Context(m, n, nl, variant=variant, nblocks=nblocks, max_sweeps=64, want_x=want_x, world_size=world,
                       rank=r, nccl_id=lid, stream=streams[r], **kw) for r in range(world)]
    for c in ctxs:
        load(c, P)
    res = [None] * world
    errs = []

    def run(r):
        try:
            st = ctxs[r].sweep()
            out = ctxs[r].extract()
            X = ctxs[r].extract_x() if want_x else None
            res[r] = (st, out, X, ctxs[r].extract_local() if local else None)
        except Exception as e:  # noqa: BLE001 -- reported below
            errs.append((r, repr(e)))

    th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=900)
    assert not any(t.is_alive() for t in th), "a rank hung"
    for c in ctxs:
        c.close()
    assert not errs, errs
    return res


def assert_same(a, b):
    sta, (la, fa, ga, Za), Xa = a[:3]
    stb, (lb, fb, gb, Zb), Xb = b[:3]
    assert sta["sweeps"] == stb["sweeps"]
    assert sta["converged"] == stb["converged"] == 1
    assert sta["transforms_all"] == stb["transforms_all"]
    assert sta["transforms_big"] == stb["transforms_big"]
    for x, y in ((la, lb), (fa, fb), (ga, gb), (Za, Zb)):
        np.testing.assert_array_equal(x, y)
    if Xa is not None:
        np.testing.assert_array_equal(Xa, Xb)


@pytest.mark.parametrize("world,nblocks", [(2, 8), (2, 12), (4, 8), (4, 16), (8, 16)])
def test_loopback_ranks_bitwise_equal_single(gh, world, nblocks):
    P = inputs.known_hyperbolic(21, 400, 256, 0.4)
    ref = single(gh, P, nblocks, False)
    res = multi(gh, P, nblocks, world, False, f"t{world}_{nblocks}")
    for r in range(world):
        assert_same(res[r], ref)
    # and the eigenvalues are the constructed ones
    lam = np.sort(ref[1][0])
    assert float(np.max(np.abs(lam - np.sort(P.lam_true)) / np.abs(np.sort(P.lam_true)))) <= 1e-9


@pytest.mark.parametrize("n,nblocks,world", [(191, 8, 2), (250, 12, 3), (129, 6, 3)])
def test_loopback_odd_and_ragged(gh, n, nblocks, world):
    """Odd n (bordered to even order, Sec 6.3.2) and ragged block widths (w and w-1)."""
    P = inputs.known_hyperbolic(24 + n, n + 77, n, 0.4)
    ref = single(gh, P, nblocks, False)
    res = multi(gh, P, nblocks, world, False, f"odd{n}_{world}")
    for r in range(world):
        assert_same(res[r], ref)


def test_loopback_fb(gh):
    """FB (inner sweeps to convergence) with two ranks."""
    P = inputs.known_hyperbolic(23, 320, 192, 0.4)
    ref = single(gh, P, 12, False, "fb")
    res = multi(gh, P, 12, 2, False, "fb2", "fb")
    for r in range(2):
        assert_same(res[r], ref)


def test_loopback_want_x(gh):
    """NEXT-1 with several ranks: W^T block columns travel with F, G, Z; X = Z^{-1}."""
    P = inputs.known_hyperbolic(22, 300, 192, 0.5)
    ref = single(gh, P, 12, True)
    res = multi(gh, P, 12, 3, True, "x3")
    for r in range(3):
        assert_same(res[r], ref)
    lam, sf, sg, Z = ref[1]
    err = np.linalg.norm(ref[2] @ Z - np.eye(Z.shape[0])) / np.sqrt(Z.shape[0])
    assert err <= 1e-9


def test_loopback_illcond_tall(gh):
    """Config-3 recipe at reduced size (Phase 1 on ill-conditioned atoms, S singular values
    1 .. 1e-12, tall 2 N_A N_L x N_G factors), two and four ranks."""
    at = inputs.illcond_atoms(33, 4, 49, 256, smin=1e-6)
    ref = single(gh, at, 8, False)
    for world in (2, 4):
        res = multi(gh, at, 8, world, False, f"c3s{world}")
        for r in range(world):
            assert_same(res[r], ref)


def test_loopback_resumed_sweeps(gh):
    """Multi-rank resume: each rank calls ghsvd_sweep repeatedly with C_max = 2 (the block
    columns are back with their step-0 owners after every sweep) -- bitwise equal to the
    one-rank single-call solve."""
    import torch
    import warnings
    P = inputs.known_hyperbolic(25, 320, 192, 0.4)
    m, n = P.F.shape
    ref = single(gh, P, 12, False)
    lid = gh.loopback_id("resume3")
    ctxs = [gh.Context(m, n, variant="bo", nblocks=12, max_sweeps=2, world_size=3, rank=r, nccl_id=lid,
                       stream=torch.cuda.Stream()) for r in range(3)]
    for c in ctxs:
        c.set_factors(P.F, P.J, P.G)
    res, errs = [None] * 3, []

    def run(r):
        try:
            total = 0
            with warnings.catch_warnings():
                warnings.simplefilter("ignore")
                for _ in range(40):
                    st = ctxs[r].sweep()
                    total += st["sweeps"]
                    if st["converged"]:
                        break
            res[r] = (total, ctxs[r].extract())
        except Exception as e:  # noqa: BLE001
            errs.append(repr(e))

    th = [threading.Thread(target=run, args=(r,)) for r in range(3)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    for c in ctxs:
        c.close()
    assert not errs, errs
    for total, (lam, sf, sg, Z) in res:
        assert total == ref[0]["sweeps"]
        np.testing.assert_array_equal(lam, ref[1][0])
        np.testing.assert_array_equal(Z, ref[1][3])


@pytest.mark.parametrize("overlap", [False, True])
def test_loopback_exchange_modes_and_distributed_z(gh, overlap):
    """Both exchange modes (exchange_overlap 0: one grouped F, G, Z' exchange per block step
    on the context stream -- the default, one communicator; 1: the two-part exchange on two
    streams) give the one-rank result bitwise, and ghsvd_extract_local leaves Z distributed:
    every column is held by exactly one rank, bitwise equal to the one-rank Z column, with
    complete lambda / Sigma on every rank."""
    P = inputs.known_hyperbolic(21, 400, 256, 0.4)
    ref = single(gh, P, 16, False)
    world = 4
    res = multi(gh, P, 16, world, False, f"xch{int(overlap)}", local=True, exchange_overlap=overlap)
    n = P.F.shape[1]
    seen = np.zeros(n, int)
    for r in range(world):
        assert_same(res[r], ref)
        lam, sf, sg, Zl, ids = res[r][3]
        np.testing.assert_array_equal(lam, ref[1][0])
        np.testing.assert_array_equal(sf, ref[1][1])
        assert Zl.shape == (n, len(ids)) and len(ids) < n
        np.testing.assert_array_equal(Zl, ref[1][3][:, ids])
        seen[ids] += 1
    assert np.all(seen == 1)


def test_extract_local_one_rank_is_extract(gh):
    P = inputs.known_hyperbolic(22, 120, 64, 0.4)
    c = gh.Context(120, 64, variant="bo", nblocks=4)
    c.set_factors(P.F, P.J, P.G)
    c.sweep()
    lam, sf, sg, Z = c.extract()
    l2, f2, g2, Zl, ids = c.extract_local()
    c.close()
    assert list(ids) == list(range(64))
    for x, y in ((lam, l2), (sf, f2), (sg, g2), (Z, Zl)):
        np.testing.assert_array_equal(x, y)
