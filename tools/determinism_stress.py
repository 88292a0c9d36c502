"""Race detector by repetition (compute-sanitizer is unavailable on this pool): run the
same blocked / pointwise / Phase-1 problems N times and require bitwise-identical
results (every reduction in the library has a fixed order, so any difference means a
race).  usage: python tools/determinism_stress.py [N]"""
import os
import sys
import warnings

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1907_08560_b200 import build, ghsvd, inputs  # noqa: E402

warnings.simplefilter("ignore")
build.build()
N = int(sys.argv[1]) if len(sys.argv) > 1 else 10
P = inputs.known_hyperbolic(21, 600, 256, 0.5)
cases = [("bo", {}), ("bo", {"GHSVD_PIVOT_CL": "1"}), ("fb", {}), ("pointwise", {})]
bad = 0
for variant, env in cases:
    os.environ.update(env)
    ref = None
    for i in range(N):
        ctx = ghsvd.Context(600, 256, variant=variant, want_x=variant != "fb")
        ctx.set_factors(P.F, P.J, P.G)
        st = ctx.sweep()
        lam, sf, sg, Z = ctx.extract()
        X = ctx.extract_x() if variant != "fb" else None
        ctx.close()
        cur = (lam, Z, X, st["sweeps"])
        if ref is None:
            ref = cur
        elif not (np.array_equal(cur[0], ref[0]) and np.array_equal(cur[1], ref[1]) and cur[3] == ref[3] and
                  (X is None or np.array_equal(cur[2], ref[2]))):
            bad += 1
            print(f"NONDETERMINISTIC: {variant} {env} run {i}")
    for k in env:
        del os.environ[k]
    print(f"{variant} {env}: {N} runs, sweeps {ref[3]}")
at = inputs.lapw_atoms(9, 16, 49, 256, 39 / 98)
ref = None
for i in range(N):
    ctx = ghsvd.Context(2 * 16 * 49, 256, 49)
    ctx.factor(at.A, at.B, at.U, at.TAA, at.TAB, at.TBB)
    F, J, G, _ = ctx.get_factors()
    ctx.close()
    if ref is None:
        ref = (F, J, G)
    elif not all(np.array_equal(a, b) for a, b in zip((F, J, G), ref)):
        bad += 1
        print(f"NONDETERMINISTIC: phase1 run {i}")
print("phase1:", N, "runs")
# the bench's configuration: HIER block ordering over super blocks (reading R2-5), and the
# blocked Phase 2 with planned pivots (cuSOLVER ZGEQRF / own QR, column-pivoted), then BO
for kw in ({"ordering": "hier", "super_blocks": 4}, {"ordering": "level3", "super_blocks": 4}):
    ref = None
    for i in range(N):
        ctx = ghsvd.Context(600, 256, variant="bo", **kw)
        ctx.set_factors(P.F, P.J, P.G)
        st = ctx.sweep()
        cur = ctx.extract()
        ctx.close()
        if ref is None:
            ref = (cur, st["sweeps"])
        elif not (all(np.array_equal(a, b) for a, b in zip(cur, ref[0])) and st["sweeps"] == ref[1]):
            bad += 1
            print(f"NONDETERMINISTIC: bo {kw} run {i}")
    print(f"bo {kw}: {N} runs, sweeps {ref[1]}")
for rkw in ({"unblocked": False}, {"unblocked": False, "own_qr": True}, {"unblocked": False, "colpiv": True}):
    ref = None
    for i in range(N):
        ctx = ghsvd.Context(2 * 16 * 49, 256, 49, variant="bo")
        ctx.factor(at.A, at.B, at.U, at.TAA, at.TAB, at.TBB)
        ctx.reduce(**rkw)
        F, J, G, p2 = ctx.get_factors()
        st = ctx.sweep()
        lam = ctx.extract(want_z=False)[0].copy()
        ctx.close()
        cur = (F, J, G, p2, lam)
        if ref is None:
            ref = cur
        elif not all(np.array_equal(a, b) for a, b in zip(cur, ref)):
            bad += 1
            print(f"NONDETERMINISTIC: phase2 {rkw} run {i}")
    print(f"phase2 {rkw} + bo: {N} runs")
print("determinism stress:", "FAIL" if bad else "OK")
sys.exit(1 if bad else 0)
