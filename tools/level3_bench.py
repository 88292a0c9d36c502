"""Level-3 block orderings on the headline config (reading R2-5): full
config-3 BO solves on one GPU in the round-robin, LEVEL3 and HIER orderings (time, sweeps,
block steps, eigenvalues against the round-robin solve), plus the exchange counts and
bytes per sweep their multi-GPU schedules would move (exchange plans, host-only).

  python tools/level3_bench.py --out profiles/r02/level3_c3.json
"""
import argparse
import json
import os
import sys
import warnings

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1907_08560_b200 import build, ghsvd, inputs  # noqa: E402


def exchange_stats(ordering, nblk, nsup, world, m, n):
    """Per sweep: block steps after which something moves, and the bytes one rank sends."""
    nst = ghsvd.order_steps(ordering, nblk, nsup)
    w = n // nblk
    moving, blocks_sent = 0, 0
    for s in range(nst):
        snd, _ = ghsvd.exchange_plan(nblk, world, 0, s, (s + 1) % nst, ordering, nsup)
        any_move = any(ghsvd.exchange_plan(nblk, world, r, s, (s + 1) % nst, ordering, nsup)[0]
                       for r in range(world))
        moving += bool(any_move)
        blocks_sent += len(snd)
    return {"steps": nst, "exchanges": moving, "rank0_bytes_sent": blocks_sent * w * (2 * m + n) * 16}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--runs", nargs="+", default=["rr_0", "level3_4", "hier_4", "level3_8", "hier_8"])
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--reduce", action="store_true", help="Phase 2 before the sweep (configs 2, 6)")
    ap.add_argument("--out", default=os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                                  "profiles", "r02", "level3_c3.json"))
    args = ap.parse_args()
    build.build()
    warnings.simplefilter("ignore")
    import numpy as np
    kind, at = inputs.make_config(args.config, backend="torch" if args.config == 3 else "numpy")
    if kind == "atoms":
        NA, NL, NG = at.A.shape
        m, n = 2 * NA * NL, NG
    else:
        (m, n), NL = at.F.shape, 0
    import math

    def auto_nblk(ordering, nsup):   # the library's auto partition (blocked.cu auto_nblk), one GPU
        nb = (n + (n & 1) + 31) // 32
        nb += nb & 1
        if ordering != "rr":
            L = math.lcm(2, nsup if ordering == "level3" else 2 * nsup)
            nb = -(-nb // L) * L
        return nb
    nblk = auto_nblk("rr", 0)
    res = {"config": inputs.CONFIGS[args.config]["name"], "m": m, "n": n, "nblk": nblk, "reduce": args.reduce,
           "runs": {}, "exchange_plans": {}}
    lam_rr = None
    for run in args.runs:
        ordering, _, ns = run.partition("_")
        nsup = int(ns)
        ctx = ghsvd.Context(m, n, NL, variant="bo", max_sweeps=64, ordering=ordering, super_blocks=nsup,
                            detail_timing=2)
        if kind == "atoms":
            ctx.factor(at.A, at.B, at.U, at.TAA, at.TAB, at.TBB)
        else:
            ctx.set_factors(at.F, at.J, at.G)
        if args.reduce:
            ctx.reduce()
        st = ctx.sweep()
        lam, *_ = ctx.extract(want_z=False)
        ctx.close()
        lam = np.sort(lam)
        if lam_rr is None and ordering == "rr":
            lam_rr = lam
        d = float(np.max(np.abs(lam - lam_rr) / np.abs(lam_rr))) if lam_rr is not None else None
        nb = auto_nblk(ordering, nsup)
        nst = ghsvd.order_steps(ordering, nb, nsup)
        res["runs"][run] = {"ordering": ordering, "super_blocks": nsup, "nblk": nb, "sweeps": st["sweeps"],
                            "converged": st["converged"], "seconds": st["seconds"],
                            "steps_per_sweep": nst, "block_steps": nst * st["sweeps"],
                            "ms_per_block_step": 1e3 * st["seconds"] / (nst * st["sweeps"]),
                            "TFLOPs": st["alg_flops"] / st["seconds"] / 1e12,
                            "max_rel_lambda_vs_rr": d, "big_per_sweep": st["big_per_sweep"]}
        print(run, {k: v for k, v in res["runs"][run].items() if k != "big_per_sweep"}, flush=True)
    for world in (2, 4, 8):
        for ordering in ("rr", "level3", "hier"):
            nsup = 0 if ordering == "rr" else 2 * world
            nb = -(-nblk // (4 * world)) * 4 * world
            res["exchange_plans"][f"{ordering}_P{world}"] = exchange_stats(ordering, nb, nsup, world, m, n)
    print(json.dumps(res["exchange_plans"], indent=1))
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    json.dump(res, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
