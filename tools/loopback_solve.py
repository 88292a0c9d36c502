"""Multi-rank blocked solve of a BASELINE config on ONE GPU through the loopback transport
(include/ghsvd.h, nccl_id), checked bitwise against the one-rank solve.

  python tools/loopback_solve.py --config 4 --world 8

Each of the `world` ranks is a context of this process with full-size buffers (as on a
real multi-GPU run), driven by its own host thread; the block columns move by device
copies.  The ranks share the GPU, so the times printed are NOT multi-GPU times -- the
point is that the P-rank schedule reproduces the one-rank eigenvalues and sweep count.
"""
import argparse
import json
import os
import sys
import threading
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--world", type=int, default=2)
    ap.add_argument("--max-sweeps", type=int, default=64)
    ap.add_argument("--overlap", type=int, default=0, help="exchange_overlap of the P-rank run (0: one grouped exchange)")
    ap.add_argument("--ordering", default="rr", help="rr | level3 | hier (block ordering, csrc/ordering.h)")
    ap.add_argument("--super-blocks", type=int, default=0, help="super blocks of level3 / hier (0: 2 * world)")
    args = ap.parse_args()
    import torch
    from paper_1907_08560_b200 import build, ghsvd, inputs
    build.build()
    kind, at = inputs.make_config(args.config, backend="torch")
    assert kind == "atoms"
    NA, NL, NG = at.A.shape
    m, n = 2 * NA * NL, NG
    # the SAME ordering and super blocks on one rank and on P ranks (bitwise comparison)
    nsup = 0 if args.ordering == "rr" else (args.super_blocks or 2 * args.world)

    def make(world, rank, lid, stream):
        c = ghsvd.Context(m, n, NL, variant="bo", max_sweeps=args.max_sweeps, world_size=world, rank=rank,
                          nccl_id=lid, stream=stream, exchange_overlap=bool(args.overlap) and world > 1,
                          ordering=args.ordering, super_blocks=nsup)
        c.factor(at.A, at.B, at.U, at.TAA, at.TAB, at.TBB)
        return c

    # one rank
    c = make(1, 0, None, torch.cuda.Stream())
    t0 = time.perf_counter()
    st1 = c.sweep()
    t1 = time.perf_counter() - t0
    lam1 = c.extract(want_z=False)[0].copy()
    c.close()
    del c
    torch.cuda.empty_cache()
    # P ranks
    lid = ghsvd.loopback_id(f"cfg{args.config}_w{args.world}_x{args.overlap}_{args.ordering}")
    ctxs = [make(args.world, r, lid, torch.cuda.Stream()) for r in range(args.world)]
    res, errs = [None] * args.world, []

    def run(r):
        try:
            st = ctxs[r].sweep()
            res[r] = (st, ctxs[r].extract(want_z=False)[0].copy())
        except Exception as e:  # noqa: BLE001
            errs.append(repr(e))

    th = [threading.Thread(target=run, args=(r,)) for r in range(args.world)]
    t0 = time.perf_counter()
    for t in th:
        t.start()
    for t in th:
        t.join()
    tP = time.perf_counter() - t0
    for c in ctxs:
        c.close()
    ok = not errs and all(r is not None and r[0]["sweeps"] == st1["sweeps"] and np.array_equal(r[1], lam1)
                          for r in res)
    out = {"config": args.config, "m": m, "n": n, "world": args.world, "exchange_overlap": args.overlap,
           "ordering": args.ordering, "super_blocks": nsup, "one_rank": {
        "sweeps": st1["sweeps"], "converged": st1["converged"], "sweep_seconds": st1["seconds"], "wall_s": t1},
        "loopback": {"per_rank_sweep_seconds": [r[0]["seconds"] for r in res if r], "wall_s": tP,
                     "sweeps": [r[0]["sweeps"] for r in res if r], "errors": errs},
        "bitwise_equal": bool(ok),
        "note": "loopback ranks share one GPU: times are not multi-GPU times"}
    print(json.dumps(out))
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
