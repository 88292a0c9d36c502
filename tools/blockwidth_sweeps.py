"""Oracle sweep counts of the blocked BO variant by block width w (NEXT-2's question: would
a third blocking level -- block pivots of order 128, w = 64 -- save sweeps?).  Oracle only
(or_hz_blocked, Sec 6.4), on the config-3 recipe at n = 1024 (the stored-reference analog)
and on a dataset-C-shaped GSVD pencil (J = I, Hermitian factors with U(0, 1) spectra,
n = 1024).

  OMP_NUM_THREADS=8 python tools/blockwidth_sweeps.py --out profiles/r02/blockwidth_sweeps.json
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
    ap.add_argument("--widths", type=int, nargs="+", default=[16, 32, 64])
    ap.add_argument("--cases", nargs="+", default=["illcond_16_49_1024_s31", "datasetC_1024_s5"])
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02", "blockwidth_sweeps.json"))
    args = ap.parse_args()
    import oracle
    from paper_1907_08560_b200 import inputs
    cases = {}
    if "illcond_16_49_1024_s31" in args.cases:
        at = inputs.illcond_atoms(31, 16, 49, 1024)
        cases["illcond_16_49_1024_s31"] = oracle.factor(at.A, at.B, at.U, at.TAA, at.TAB, at.TBB)
    if "datasetC_1024_s5" in args.cases:
        # (seed 7 draws an eigenvalue of F small enough that a block pivot is numerically
        # singular: the stop the paper prescribes)
        P = inputs.dataset_c(5, 1024)
        cases["datasetC_1024_s5"] = (P.F, P.J, P.G)
    res = json.load(open(args.out)) if os.path.exists(args.out) else {}
    res.update({"what": "or_hz_blocked BO sweeps by block width w (nblk = 2 ceil(n / 2w)), C_max 64"})
    res.setdefault("cases", {})
    for name, (F, J, G) in cases.items():
        n = F.shape[1]
        res["cases"][name] = {}
        for w in args.widths:
            nblk = 2 * ((n + 2 * w - 1) // (2 * w))
            t = time.time()
            _, _, _, st = oracle.hz_blocked(F, J, G, nblk, inner_sweeps=1, cmax=64)
            res["cases"][name][f"w{w}"] = {"nblk": nblk, "sweeps": st["sweeps"], "converged": st["converged"],
                                           "seconds": time.time() - t}
            print(name, w, res["cases"][name][f"w{w}"], flush=True)
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    json.dump(res, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
