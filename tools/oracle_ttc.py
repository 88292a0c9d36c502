"""Measured oracle time-to-converge for the small BASELINE configs ("Report
time-to-converge, sweeps and pairs visited/s for configs 0-3" for the oracle on the host
cores).  Oracle only: inputs.make_config -> oracle Phase 1 (and Phase 2 where the recipe
has it) -> oracle.hz_pointwise (Alg. 2) timed end to end, once per config.  Config 3's
measured full solve is the stored reference tests/golden/c3_oracle_pointwise.json.

  OMP_NUM_THREADS=8 python tools/oracle_ttc.py --configs 0 1 2 --out profiles/r02/oracle_ttc.json
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
    ap.add_argument("--configs", type=int, nargs="+", default=[0, 1, 2])
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02", "oracle_ttc.json"))
    args = ap.parse_args()
    import importlib.util
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    b = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(b)
    import oracle
    from paper_1907_08560_b200 import inputs
    cores = b._cores()
    # untimed warm-up: the first OpenMP region of the process starts the thread pool (~0.8 s)
    k0, p0 = inputs.make_config(0)
    oracle.hz_pointwise(*b.oracle_factors(k0, p0, 0), cmax=1, nthreads=cores)
    res = {"cpu_model": b._cpu_model(), "threads": cores, "what": "oracle.hz_pointwise to convergence (C_max 64), "
           "timed end to end on the oracle's own starting factors", "configs": {}}
    for c in args.configs:
        kind, payload = inputs.make_config(c, backend="numpy")
        t = time.perf_counter()
        F, J, G = b.oracle_factors(kind, payload, c)
        t_pre = time.perf_counter() - t
        m, n = F.shape
        t = time.perf_counter()
        _, _, _, st = oracle.hz_pointwise(F, J, G, cmax=64, nthreads=cores)
        tt = time.perf_counter() - t
        res["configs"][inputs.CONFIGS[c]["name"]] = {
            "m": m, "n": n, "sweeps": st["sweeps"], "converged": st["converged"], "seconds": tt,
            "pairs_visited_per_s": st["pairs_visited"] / tt, "transforms_per_s": st["transforms_all"] / tt,
            "phase12_seconds": t_pre}
        print(c, res["configs"][inputs.CONFIGS[c]["name"]], flush=True)
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    json.dump(res, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
