"""Write a stored ORACLE reference for a BASELINE config (SURVEY.md Sec 8(c) pins table:
"Config 3 accuracy ... At full size: oracle vs GPU, both GHSVD, <= 1e-6 per BASELINE";
VERDICT r1 "Next round" item 1).

Calls only ``oracle/`` and the seeded input generator (``inputs``, which holds no
method arithmetic).  Nothing here touches the CUDA path:

  1. atoms of the config by ``inputs.make_config(cfg, backend="numpy")`` (host QRs);
  2. Phase 1 by ``oracle.factor`` (Alg. 1, eqs 4.1-4.3);
  3. Phase 3 to convergence by ``oracle.hz_pointwise`` (Alg. 2) or
     ``oracle.hz_blocked`` (Sec. 6.4, BO with the GPU's auto partition);
  4. outputs by ``oracle.extract``.

Output ``tests/golden/c<cfg>_oracle_<variant>.npz`` (lambda in column order, Sigma_F,
Sigma_G) and ``.json`` (input fingerprint, sweeps and counters, wall time, host CPU model
and thread count).  The GPU test re-generates the atoms, checks the fingerprint, and
compares its converged eigenvalues with these per eigenvalue at the north-star tolerance.

  OMP_NUM_THREADS=8 python tools/make_oracle_reference.py --config 3 --variant pointwise
"""
import argparse
import hashlib
import json
import os
import platform
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--illcond", type=str, default="",
                    help="NA,NL,NG,seed: a scaled-down config-3 analog (inputs.illcond_atoms) instead of --config")
    ap.add_argument("--variant", choices=["pointwise", "bo", "dense"], default="pointwise",
                    help="dense: oracle.pencil_eigvals (form H, S; ZHEGVD; PAPER.md:818-836), "
                         "for well-conditioned S only (config 4)")
    ap.add_argument("--nblk", type=int, default=0, help="BO block columns (0: 2*ceil(n/64), the GPU auto partition)")
    ap.add_argument("--cmax", type=int, default=64)
    ap.add_argument("--threads", type=int, default=0)
    ap.add_argument("--out", default=os.path.join(ROOT, "tests", "golden"))
    args = ap.parse_args()

    import oracle
    from paper_1907_08560_b200 import inputs

    t0 = time.time()
    if args.illcond:
        NA, NL, NG, seed = (int(v) for v in args.illcond.split(","))
        at = inputs.illcond_atoms(seed, NA, NL, NG)
        name = f"illcond_{NA}_{NL}_{NG}_s{seed}"
    else:
        kind, at = inputs.make_config(args.config, backend="numpy")
        name = f"c{args.config}"
    t_gen = time.time() - t0
    fp = inputs.fingerprint(at)
    raw = hashlib.sha256()
    atoms = hasattr(at, "TAA")
    for arr in (("A", "B", "U", "TAA", "TAB", "TBB") if atoms else ("F", "J", "G")):
        raw.update(np.ascontiguousarray(getattr(at, arr)).tobytes())

    t0 = time.time()
    if atoms:
        F, J, G = oracle.factor(at.A, at.B, at.U, at.TAA, at.TAB, at.TBB)
    else:
        # a pencil given directly (config 5, dataset C: J = I, n even): the sweep's factors
        # as given (no row sort needed with J = I, no border with n even)
        assert np.all(at.J == 1) and at.F.shape[1] % 2 == 0, "pencil references: J = I, even n"
        F, J, G = np.asfortranarray(at.F), np.asarray(at.J, np.int8), np.asfortranarray(at.G)
    t_factor = time.time() - t0
    del at
    m, n = F.shape
    nblk = args.nblk or 2 * ((n + 63) // 64)
    threads = args.threads or len(os.sched_getaffinity(0))
    print(f"{name}: m={m} n={n} variant={args.variant} threads={threads} "
          f"(gen {t_gen:.1f} s, factor {t_factor:.1f} s)", flush=True)

    t0 = time.time()
    if args.variant == "dense":
        lam = oracle.pencil_eigvals(F, J, G)
        t_sweep = time.time() - t0
        # kappa(S) of this pencil, the justification for the dense route (its error ~ eps kappa(S) ||H||)
        sev = np.linalg.eigvalsh(G.conj().T @ G)
        st = {"converged": True, "sweeps": None, "kappa_S": float(sev[-1] / sev[0]),
              "lam_abs_min": float(np.abs(lam).min()), "lam_abs_max": float(np.abs(lam).max()),
              "negative": int((lam < 0).sum())}
        print(f"dense: {t_sweep:.1f} s, kappa(S) = {st['kappa_S']:.3g}", flush=True)
        stem = os.path.join(args.out, f"{name}_oracle_dense")
        np.savez_compressed(stem + ".npz", lam=lam)
        meta = {
            "about": "Oracle-only reference (tools/make_oracle_reference.py --variant dense): "
                     "inputs.make_config(numpy) -> oracle.factor -> oracle.pencil_eigvals (H = F^*JF, "
                     "S = G^*G formed, ZHEGVD). No value comes from the CUDA path.",
            "cite": "PAPER.md:818-836 (Sec 4.5, the alternative way forward; valid for well-conditioned S); "
                    "SURVEY.md Sec 8(c) pins table (config 4: oracle run once, cached by an input hash)",
            "config": name, "m": m, "n": n, "variant": "dense", "stats": st,
            "seconds_solve": t_sweep, "seconds_factor": t_factor, "seconds_generate": t_gen,
            "threads": threads, "cpu_model": cpu_model(), "host_cores": os.cpu_count(),
            "inputs_sha256": raw.hexdigest(), "fingerprint": fp, "lam_file": os.path.basename(stem + ".npz"),
        }
        with open(stem + ".json", "w") as f:
            json.dump(meta, f, indent=1)
        print("wrote", stem + ".npz", stem + ".json")
        return
    if args.variant == "pointwise":
        Fc, Gc, Zp, st = oracle.hz_pointwise(F, J, G, cmax=args.cmax, nthreads=threads)
    else:
        Fc, Gc, Zp, st = oracle.hz_blocked(F, J, G, nblk, inner_sweeps=1, cmax=args.cmax, nthreads=threads)
    t_sweep = time.time() - t0
    lam, sf, sg, _ = oracle.extract(Fc, J, Gc, Zp)
    print(f"sweeps={st['sweeps']} converged={st['converged']} seconds={t_sweep:.1f}", flush=True)

    stem = os.path.join(args.out, f"{name}_oracle_{args.variant}")
    np.savez_compressed(stem + ".npz", lam=lam, sigma_f=sf, sigma_g=sg)
    meta = {
        "about": "Oracle-only reference (tools/make_oracle_reference.py): inputs.make_config(numpy) -> "
                 "oracle.factor -> oracle.hz_%s -> oracle.extract. No value comes from the CUDA path." % (
                     "pointwise" if args.variant == "pointwise" else "blocked (BO)"),
        "cite": "SURVEY.md Sec 8(c) pins table (config 3: oracle vs GPU <= 1e-6); PAPER.md:2189-2201 (Sec 7)",
        "config": name, "m": m, "n": n, "variant": args.variant,
        "nblk": nblk if args.variant == "bo" else None, "cmax": args.cmax,
        "stats": st, "seconds_sweep": t_sweep, "seconds_factor": t_factor, "seconds_generate": t_gen,
        "threads": threads, "cpu_model": cpu_model(), "host_cores": os.cpu_count(),
        "inputs_sha256": raw.hexdigest(), "fingerprint": fp,
        "lam_file": os.path.basename(stem + ".npz"),
    }
    with open(stem + ".json", "w") as f:
        json.dump(meta, f, indent=1)
    print("wrote", stem + ".npz", stem + ".json")


if __name__ == "__main__":
    main()
