"""Oracle sweep counts of the blocked BO variant by block ordering (reading R2-5, the
Level-3 orderings of PAPER.md:1815-1824 Sec 6.4): round-robin vs LEVEL3 (recursive BO
over nsup super blocks) vs HIER (every block pair once, grouped by super pair).  Oracle
only (or_hz_blocked_ord), on the config-3 recipe at n = 1024 and a dataset-C-shaped GSVD
pencil at n = 1024, block width 32 (nblk = 32) as on the GPU.

  OMP_NUM_THREADS=8 python tools/ordering_sweeps.py --out profiles/r02/ordering_sweeps.json
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", nargs="+", default=["illcond_16_49_1024_s31", "datasetC_1024_s5"])
    ap.add_argument("--runs", nargs="+", default=["rr", "l3_4", "l3_8", "hier_4", "hier_8"])
    ap.add_argument("--nblk", type=int, default=32)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02", "ordering_sweeps.json"))
    args = ap.parse_args()
    import oracle
    from paper_1907_08560_b200 import inputs
    cases = {}
    if "illcond_16_49_1024_s31" in args.cases:
        at = inputs.illcond_atoms(31, 16, 49, 1024)
        cases["illcond_16_49_1024_s31"] = oracle.factor(at.A, at.B, at.U, at.TAA, at.TAB, at.TBB)
    if "datasetC_1024_s5" in args.cases:
        P = inputs.dataset_c(5, 1024)
        cases["datasetC_1024_s5"] = (P.F, P.J, P.G)
    kinds = {"rr": oracle.ORDER_RR, "l3": oracle.ORDER_LEVEL3, "hier": oracle.ORDER_HIER}
    res = json.load(open(args.out)) if os.path.exists(args.out) else {}
    res.update({"what": "or_hz_blocked_ord BO sweeps by block ordering, nblk = %d, C_max 64" % args.nblk})
    res.setdefault("cases", {})
    for name, (F, J, G) in cases.items():
        res["cases"].setdefault(name, {})
        for run in args.runs:
            kind, _, ns = run.partition("_")
            nsup = int(ns) if ns else 0
            t = time.time()
            _, _, _, st = oracle.hz_blocked(F, J, G, args.nblk, inner_sweeps=1, cmax=64, ordering=kinds[kind],
                                            nsup=nsup)
            nst = oracle.order_steps(kinds[kind], args.nblk, nsup)
            res["cases"][name][run] = {"nsup": nsup, "steps_per_sweep": nst, "sweeps": st["sweeps"],
                                       "block_steps": nst * st["sweeps"], "converged": st["converged"],
                                       "big_per_sweep": st["big_per_sweep"][:st["sweeps"]],
                                       "seconds": time.time() - t}
            print(name, run, {k: v for k, v in res["cases"][name][run].items() if k != "big_per_sweep"}, flush=True)
            os.makedirs(os.path.dirname(args.out), exist_ok=True)
            json.dump(res, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
