"""World-size-2 CPU test of the multi-GPU blocked schedule (Sec 6.4.3).

Two processes (torch.distributed, gloo, 127.0.0.1) play the two GPU ranks: each owns the
round-robin slots libghsvd assigns to it (ghsvd_block_owner), processes only its block
pairs (block-pivot numerics from the oracle, standing in for the device kernels), moves the
block columns of F, G, Z exactly as ghsvd_exchange_plan prescribes (gloo send/recv standing
in for ncclSend/ncclRecv) and all-reduces the counters once per sweep.  The result must be
BITWISE equal to the single-process blocked run with the same partition and ordering --
any missing/stale block column, wrong owner or wrong stop decision breaks equality.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rr(n, s, k):
    if k == 0:
        a, b = n - 1, s
    else:
        a, b = (s + k) % (n - 1), (s - k) % (n - 1)
    return min(a, b), max(a, b)


def _worker(rank, world, port, nblk, out_q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    from paper_1907_08560_b200 import ghsvd, inputs
    P = inputs.known_hyperbolic(14, 96, 64, 0.4)
    m, n = P.F.shape
    F = np.asfortranarray(P.F.copy())
    G = np.asfortranarray(P.G.copy())
    Z = np.asfortranarray(np.eye(n, dtype=np.complex128))
    start, width = oracle.block_partition(n, nblk)
    K = nblk // 2 // world
    sweeps = 0
    for sw in range(30):
        cnt = torch.zeros(2, dtype=torch.int64)
        for s in range(nblk - 1):
            for k in range(rank * K, (rank + 1) * K):
                bp, bq = _rr(nblk, s, k)
                assert ghsvd.block_owner(nblk, world, s, bp) == rank == ghsvd.block_owner(nblk, world, s, bq)
                a, b = oracle.block_pair(F, P.J, G, Z, start[bp], width[bp], start[bq], width[bq])
                cnt[0] += a
                cnt[1] += b
            s_next = (s + 1) % (nblk - 1)
            sends, recvs = ghsvd.exchange_plan(nblk, world, rank, s, s_next)
            reqs, bufs = [], []
            for blk, peer in sends:
                c0, w = int(start[blk]), int(width[blk])
                for X in (F, G, Z):
                    t = torch.from_numpy(np.ascontiguousarray(X[:, c0:c0 + w]))
                    bufs.append(t)
                    reqs.append(dist.isend(t, peer))
            incoming = []
            for blk, peer in recvs:
                c0, w = int(start[blk]), int(width[blk])
                for X in (F, G, Z):
                    t = torch.empty((X.shape[0], w), dtype=torch.complex128)
                    incoming.append((X, c0, w, t))
                    reqs.append(dist.irecv(t, peer))
            for r in reqs:
                r.wait()
            for X, c0, w, t in incoming:
                X[:, c0:c0 + w] = t.numpy()
        dist.all_reduce(cnt)                      # stands in for the per-sweep ncclAllReduce
        sweeps = sw + 1
        if int(cnt[1]) == 0:
            break
    # collect the final owned block columns (ownership of step 0 after the last exchange)
    own = [ghsvd.block_owner(nblk, world, 0, b) for b in range(nblk)]
    for b in range(nblk):
        c0, w = int(start[b]), int(width[b])
        for X in (F, G, Z):
            t = torch.from_numpy(np.ascontiguousarray(X[:, c0:c0 + w]))
            dist.broadcast(t, src=own[b])
            X[:, c0:c0 + w] = t.numpy()
    if rank == 0:
        out_q.put((F, G, Z, sweeps))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("nblk", [8])
def test_two_rank_blocked_equals_single_process(nblk):
    from paper_1907_08560_b200 import build
    build.build()
    import oracle
    from paper_1907_08560_b200 import inputs
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, nblk, q)) for r in range(2)]
    for p in procs:
        p.start()
    F, G, Z, sweeps = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    P = inputs.known_hyperbolic(14, 96, 64, 0.4)
    Fo, Go, Zo, st = oracle.hz_blocked(P.F, P.J, P.G, nblk, inner_sweeps=1)
    assert sweeps == st["sweeps"]
    assert np.array_equal(F, Fo) and np.array_equal(G, Go) and np.array_equal(Z, Zo)


def test_exchange_plan_is_consistent():
    """Every block sent by one rank is received by its new owner from the old owner, for
    P = 2, 4, 8 and K = 1, 2, 4 block pairs per rank (the round-robin with slot
    k -> GPU k moves at most 2 block columns out of and into each GPU per block step)."""
    from paper_1907_08560_b200 import build, ghsvd
    build.build()
    for world, K in [(w, k) for w in (2, 4, 8) for k in (1, 2, 4)]:
        nblk = 2 * K * world
        for s in range(nblk - 1):
            s2 = (s + 1) % (nblk - 1)
            sent, recv = set(), set()
            for r in range(world):
                sd, rv = ghsvd.exchange_plan(nblk, world, r, s, s2)
                assert len(sd) <= 2 and len(rv) == len(sd)
                for b, peer in sd:
                    assert ghsvd.block_owner(nblk, world, s, b) == r and ghsvd.block_owner(nblk, world, s2, b) == peer
                    sent.add((b, r, peer))
                for b, peer in rv:
                    assert ghsvd.block_owner(nblk, world, s2, b) == r and ghsvd.block_owner(nblk, world, s, b) == peer
                    recv.add((b, peer, r))
            assert sent == recv
            # ownership covers each block exactly once per step
            for b in range(nblk):
                assert 0 <= ghsvd.block_owner(nblk, world, s, b) < world


def _inputs_worker(rank, world, port, cfg, out_q):
    import hashlib
    import importlib.util
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    b = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(b)
    kind, payload = b.shared_inputs(cfg, world, rank, torch.device("cpu"))
    h = hashlib.sha256()
    names = ("A", "B", "U", "TAA", "TAB", "TBB") if kind == "atoms" else ("F", "J", "G")
    for k in names:
        h.update(np.ascontiguousarray(getattr(payload, k)).tobytes())
    out_q.put((rank, kind, h.hexdigest()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("cfg", [0, 1])
def test_bench_inputs_broadcast_identical(cfg):
    """bench.py's multi-rank input path: rank 0 generates the seeded inputs once and
    broadcasts them; every rank holds bitwise the inputs a single process generates."""
    import hashlib
    from paper_1907_08560_b200 import inputs
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_inputs_worker, args=(r, 2, port, cfg, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    kind, payload = inputs.make_config(cfg, backend="numpy")
    h = hashlib.sha256()
    names = ("A", "B", "U", "TAA", "TAB", "TBB") if kind == "atoms" else ("F", "J", "G")
    for k in names:
        h.update(np.ascontiguousarray(getattr(payload, k)).tobytes())
    assert {g[2] for g in got} == {h.hexdigest()} and {g[1] for g in got} == {kind}
