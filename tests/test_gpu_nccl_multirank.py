"""The multi-GPU blocked sweep over REAL NCCL (Sec 6.4.3,
lines 1974-2040): P processes, one GPU each, ncclSend/ncclRecv of block columns per block
step and one allreduce of the counters per sweep.  The result must be bitwise equal to
the one-rank solve with the same partition (the per-pair arithmetic and the Gram split
do not depend on the rank count).  Needs >= 2 visible GPUs; skipped otherwise (the same
schedule is covered on one GPU by the loopback transport, test_gpu_multirank_loopback.py,
and on CPU by the gloo emulation, test_multirank_gloo.py)."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ngpus():
    import torch
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, overlap, out_q):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    from paper_1907_08560_b200 import ghsvd, inputs
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    idt = torch.zeros(128, dtype=torch.uint8, device=dev)
    if rank == 0:
        idt.copy_(torch.frombuffer(bytearray(ghsvd.nccl_unique_id()), dtype=torch.uint8))
    dist.broadcast(idt, 0)
    P = inputs.known_hyperbolic(21, 400, 256, 0.4)
    stream = torch.cuda.Stream(dev)
    c = ghsvd.Context(400, 256, variant="bo", nblocks=16, max_sweeps=64, device=rank, stream=stream,
                      world_size=world, rank=rank, nccl_id=bytes(idt.cpu().numpy().tobytes()),
                      exchange_overlap=overlap)
    with torch.cuda.stream(stream):
        c.set_factors(P.F, P.J, P.G)
        st = c.sweep()
        lam, sf, sg, Z = c.extract()
        _, _, _, Zl, ids = c.extract_local()
    c.close()
    out_q.put((rank, st["sweeps"], lam, Z, Zl, ids))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("overlap", [False, True])
def test_nccl_ranks_bitwise_equal_single(world, overlap):
    if _ngpus() < world:
        pytest.skip(f"needs {world} GPUs, {_ngpus()} visible")
    import torch.multiprocessing as mp
    from paper_1907_08560_b200 import build, ghsvd, inputs
    build.build()
    P = inputs.known_hyperbolic(21, 400, 256, 0.4)
    c = ghsvd.Context(400, 256, variant="bo", nblocks=16, max_sweeps=64)
    c.set_factors(P.F, P.J, P.G)
    st1 = c.sweep()
    lam1, _, _, Z1 = c.extract()
    c.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, overlap, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = sorted((q.get(timeout=600) for _ in range(world)), key=lambda g: g[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    seen = np.zeros(256, int)
    for rank, sweeps, lam, Z, Zl, ids in got:
        assert sweeps == st1["sweeps"]
        np.testing.assert_array_equal(lam, lam1)
        np.testing.assert_array_equal(Z, Z1)
        np.testing.assert_array_equal(Zl, Z1[:, ids])
        seen[ids] += 1
    assert np.all(seen == 1)
