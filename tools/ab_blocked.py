"""A/B timing of blocked-sweep variants on a BASELINE config (exploration tool).

  python tools/ab_blocked.py [--config 3] [--sweeps 0] [--reps 2] VARIANT ...

VARIANT is `name:k=v,k=v` with Context keyword overrides (schedule=64, groups=2, ...),
or `name` alone for the defaults.  Each variant solves the same factors (Phase 1 once,
exported, then set_factors per run); prints per-variant device seconds, sweeps, s/sweep
and (with --trace) the launch-timeline summary of the first sweep.
"""
import argparse
import json
import os
import subprocess
import sys
import warnings

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--sweeps", type=int, default=0, help="C_max (0: to convergence, 64)")
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--trace", action="store_true")
    ap.add_argument("variants", nargs="*", default=["default"])
    args = ap.parse_args()
    import numpy as np
    import torch
    from paper_1907_08560_b200 import build, ghsvd, inputs
    build.build()
    warnings.simplefilter("ignore")
    kind, at = inputs.make_config(args.config, backend="torch")
    NA, NL, NG = at.A.shape
    m, n = 2 * NA * NL, NG
    c = ghsvd.Context(m, n, NL, variant="bo")
    c.factor(at.A, at.B, at.U, at.TAA, at.TAB, at.TBB)
    F, J, G, _ = c.get_factors()
    c.close()
    cmax = args.sweeps or 64
    ref = None
    for v in args.variants:
        name, _, kv = v.partition(":")
        kw = {}
        for item in filter(None, kv.split(",")):
            k, _, val = item.partition("=")
            kw[k] = int(val)
        times = []
        for rep in range(args.reps):
            tp = f"/tmp/ab_{name}.csv" if (args.trace and rep == 0) else None
            ctx = ghsvd.Context(m, n, variant="bo", max_sweeps=cmax, trace_path=tp, **kw)
            ctx.set_factors(F, J, G)
            st = ctx.sweep()
            lam = ctx.extract(want_z=False)[0].copy()
            ctx.close()
            times.append(st["seconds"])
        same = None if ref is None else bool(np.array_equal(lam, ref))
        if ref is None:
            ref = lam
        out = {"variant": name, "kw": kw, "seconds": times, "sweeps": st["sweeps"],
               "s_per_sweep": min(times) / st["sweeps"], "bitwise_same_lambda_as_first": same}
        print(json.dumps(out), flush=True)
        if args.trace:
            r = subprocess.run([sys.executable, os.path.join(os.path.dirname(__file__), "trace_summary.py"),
                                f"/tmp/ab_{name}.csv"], capture_output=True, text=True)
            print(r.stdout, flush=True)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
