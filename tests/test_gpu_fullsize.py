"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times.

Config 3 (10368 x 4096, S condition 1e12) takes the oracle ~2 h on 8 host cores, so
  * its CONVERGED eigenvalues (BO and pointwise) are compared per eigenvalue with a stored
    oracle reference (tests/golden/c3_oracle_*.{json,npz}, written by the oracle-only
    script tools/make_oracle_reference.py from the same seeded atoms, keyed by an input
    fingerprint) at the north-star ill-conditioned tolerance 1e-6;
  * elementwise on the first step / block step against the oracle run on the same
    factors, for sampled pairs, and
  * at convergence through properties that hold at any size: residual
    ||Hx - lambda Sx|| / ((||F||^2 + ||G||^2) ||x||) <= 1e-12 n for sampled eigenpairs
    (H, S never formed: Hx = F^*(J(Fx))), Sigma_F^2 + Sigma_G^2 = 1, G's columns
    orthonormal after normalisation.
Config 2 (LAPW 1568 x 1024 -> Phase 2 -> 1024^2) runs end to end against the oracle.
Config 4 (30976 x 8192): the first block step elementwise against oracle.block_pair on
the oracle's own Phase-1 factors (set_factors); convergence with residuals, and the converged
eigenvalues against a stored dense oracle reference (oracle.pencil_eigvals, PAPER.md:818-836;
S is well conditioned there) at 1e-9.
"""
import json
import os

import numpy as np
import pytest

import oracle
from paper_1907_08560_b200 import inputs

pytestmark = pytest.mark.gpu
EPS = oracle.EPS
# dataset C: the north star's well-conditioned tolerance
C5_TOL = 1e-9


@pytest.fixture(scope="module")
def gh():
    from paper_1907_08560_b200 import build, ghsvd
    build.build()
    return ghsvd


GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def c3():
    # host (numpy) generation: the stored oracle reference was computed on these atoms
    kind, at = inputs.make_config(3, backend="numpy")
    return at


def _stored_c3(variant):
    stem = os.path.join(GOLD, f"c3_oracle_{variant}")
    if not os.path.exists(stem + ".json"):
        pytest.fail(f"missing stored oracle reference {stem}.json (tools/make_oracle_reference.py)")
    return json.load(open(stem + ".json")), np.load(stem + ".npz")["lam"]


def _relerr(a, b):
    a, b = np.sort(np.asarray(a)), np.sort(np.asarray(b))
    return float(np.max(np.abs(a - b) / np.abs(b)))


_C3_LAM = {}   # eigenvalues of the bench-configuration solve, reused by later tests


def _ctx_c3(gh, at, **kw):
    NA, NL, NG = at.A.shape
    ctx = gh.Context(2 * NA * NL, NG, NL, **kw)
    ctx.factor(at.A, at.B, at.U, at.TAA, at.TAB, at.TBB)
    return ctx


@pytest.fixture(scope="module")
def c3_oracle_factors(c3):
    """The oracle's own Phase 1 (Alg. 1) of the config-3 atoms; these go to the device by
    set_factors, so no oracle input comes from the CUDA path.  The device keeps F's rows
    J-sorted (+ first, stably): row i there is row perm[i] here; G's rows stay as given."""
    F, J, G = oracle.factor(c3.A, c3.B, c3.U, c3.TAA, c3.TAB, c3.TBB)
    return F, J, G, np.argsort(-J, kind="stable")


def test_c3_pointwise_first_step_matches_oracle(gh, c3_oracle_factors):
    F, J, G, perm = c3_oracle_factors
    m, n = F.shape
    ctx = gh.Context(m, n)
    ctx.set_factors(F, J, G)
    a_g, b_g = ctx.run_steps(0, 1)
    Fg, Gg, Zg = ctx.transformed(m, n)
    ctx.close()
    Fo, Go, Zo, a, b = oracle.hz_steps(F, J, G, np.eye(n, dtype=complex), 0, 1)
    assert (a_g, b_g) == (a, b)
    # Reduction order differs (tree over J-sorted rows vs sequential over the original rows,
    # m = 10368) and the 2x2 transform amplifies Gram perturbations by ~kappa of the pair's S
    # block (S has condition 1e12 here): 1e-10 relative per column (measured 2.5e-12).
    cols = np.r_[0:64, n - 64:n]
    for X, Y in ((Fg, Fo[perm]), (Gg, Go)):
        sc = np.linalg.norm(Y[:, cols], axis=0)
        assert (np.linalg.norm(X[:, cols] - Y[:, cols], axis=0) / sc).max() < 1e-10
    assert np.abs(Zg[:, cols] - Zo[:, cols]).max() < 1e-10


def test_c3_blocked_first_block_step_matches_oracle(gh, c3_oracle_factors):
    F0, J0, G0, perm = c3_oracle_factors
    m, n = F0.shape
    ctx = gh.Context(m, n, variant="bo")
    ctx.set_factors(F0, J0, G0)
    ctx.run_steps(0, 1)
    Fg, Gg, Zg = ctx.transformed(m, n)
    ctx.close()
    nblk = 128                                   # the auto partition for n = 4096 (w = 32)
    start, width = oracle.block_partition(n, nblk)
    F = np.asfortranarray(F0.copy())
    G = np.asfortranarray(G0.copy())
    Z = np.asfortranarray(np.eye(n, dtype=complex))
    checked = []
    for k in range(0, nblk // 2, 8):             # every 8th block pair of block step 0
        p, q = oracle.rr_pair(nblk, 0, k)
        oracle.block_pair(F, J0, G, Z, start[p], width[p], start[q], width[q])
        checked += list(range(start[p], start[p] + width[p])) + list(range(start[q], start[q] + width[q]))
    # The block pivots are factored from explicitly formed Grams (Sec 6.4.2) whose condition is
    # the square of the column blocks' (G here spans 1 ... 1e-6): Gram perturbations from the
    # different summation order (~eps sqrt(m)) are amplified by kappa(S_blk).  1e-8 relative
    # per column (measured 1.7e-10); a wrong pivot / index gives O(1).
    cols = np.array(checked)
    for X, Y in ((Fg, F[perm]), (Gg, G)):
        sc = np.linalg.norm(Y[:, cols], axis=0)
        assert (np.linalg.norm(X[:, cols] - Y[:, cols], axis=0) / sc).max() < 1e-8
    assert (np.linalg.norm(Zg[:, cols] - Z[:, cols], axis=0) / np.linalg.norm(Z[:, cols], axis=0)).max() < 1e-8


def test_c3_blocked_converges_with_residuals(gh, c3):
    """The bench's configuration (BO, C_max 64) to convergence; properties at full size."""
    ctx = _ctx_c3(gh, c3, variant="bo", max_sweeps=64)
    F0, J0, G0, _ = ctx.get_factors()
    st = ctx.sweep()
    lam, sf, sg, Z = ctx.extract()
    ctx.close()
    _C3_LAM["bo"] = (lam.copy(), st["sweeps"])
    n = F0.shape[1]
    assert st["converged"] and st["big_per_sweep"][-1] == 0
    assert np.all(np.isfinite(lam))
    assert np.allclose(sf ** 2 + sg ** 2, 1.0, atol=8 * EPS)
    rng = np.random.default_rng(0)
    idx = rng.choice(n, 48, replace=False)
    x = Z[:, idx]
    nf2 = np.linalg.norm(F0) ** 2 + np.linalg.norm(G0) ** 2
    Hx = F0.conj().T @ (J0[:, None] * (F0 @ x))
    Sx = G0.conj().T @ (G0 @ x)
    res = np.linalg.norm(Hx - Sx * lam[idx][None, :], axis=0) / (nf2 * np.linalg.norm(x, axis=0))
    assert res.max() <= 1e-12 * n
    # homogeneous form (C-15): beta^2 Hx - sign alpha^2 Sx with alpha^2 + beta^2 = 1
    al2, be2 = sf[idx] ** 2, sg[idx] ** 2
    hres = np.linalg.norm(Hx * be2[None, :] - Sx * (np.sign(lam[idx]) * al2)[None, :], axis=0)
    assert (hres / (nf2 * np.linalg.norm(x, axis=0))).max() <= 1e-12 * n


def test_c3_blocked_eq71_errors(gh, c3):
    """NEXT-1 at full size: with want_x, X = Sigma Z'^{-1} and the eq (7.1) relative errors
    ||F - U Sigma_F X||_F / ||F||_F, ||G - V Sigma_G X||_F / ||G||_F on
    config 3 (products by torch on the GPU: verification only).  The paper reports
    7.98e-14 ... 8.23e-13 on its well-conditioned datasets; bound 1e-12 (measured round 1:
    eF = eG = 4.5e-14, max |ZX - I| = 6.2e-11).  Printed for the report."""
    import torch
    ctx = _ctx_c3(gh, c3, variant="bo", max_sweeps=64, want_x=True)
    F0, J0, G0, _ = ctx.get_factors()
    m, n = F0.shape
    st = ctx.sweep()
    lam, sf, sg, Z = ctx.extract()
    X = ctx.extract_x()
    Fc, Gc, _ = ctx.transformed(m, n)
    ctx.close()
    dev = "cuda"
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)   # noqa: E731
    Ft, Gt, Fct, Gct, Xt = t(F0), t(G0), t(Fc), t(Gc), t(X)
    Jt = t(J0.astype(np.float64))
    sfp = torch.sqrt(torch.abs((Fct.conj() * Fct).real.mul(Jt[:, None]).sum(0)))
    sgp = torch.linalg.norm(Gct, dim=0)
    U = Fct / sfp[None, :]
    V = Gct / sgp[None, :]
    eF = float(torch.linalg.norm(Ft - U @ (t(sf)[:, None] * Xt)) / torch.linalg.norm(Ft))
    eG = float(torch.linalg.norm(Gt - V @ (t(sg)[:, None] * Xt)) / torch.linalg.norm(Gt))
    zx = float((t(Z) @ Xt - torch.eye(n, dtype=torch.complex128, device=dev)).abs().max())
    print(f"c3 eq7.1: eF={eF:.3e} eG={eG:.3e} max|ZX-I|={zx:.3e} sweeps={st['sweeps']}")
    assert eF < 1e-12 and eG < 1e-12 and zx < 1e-8
    if "bo" in _C3_LAM:
        # a second full solve under the overlapped multi-stream schedule: bitwise the same
        # eigenvalues and sweep count (determinism; want_x only adds the W updates)
        assert np.array_equal(lam, _C3_LAM["bo"][0]) and st["sweeps"] == _C3_LAM["bo"][1]


def test_c3_two_ranks_loopback_bitwise(gh, c3):
    """The multi-GPU schedule at the bench's full size: two ranks (loopback transport, one
    GPU, two host threads; tests/test_gpu_multirank_loopback.py) reproduce the one-rank
    solve's eigenvalues and sweep count bitwise."""
    if "bo" not in _C3_LAM:
        pytest.skip("needs the one-rank solve of test_c3_blocked_converges_with_residuals")
    import threading
    import torch
    NA, NL, NG = c3.A.shape
    lid = gh.loopback_id("c3_full_2")
    ctxs = [gh.Context(2 * NA * NL, NG, NL, variant="bo", max_sweeps=64, world_size=2, rank=r, nccl_id=lid,
                       stream=torch.cuda.Stream()) for r in range(2)]
    for c in ctxs:
        c.factor(c3.A, c3.B, c3.U, c3.TAA, c3.TAB, c3.TBB)
    res, errs = [None, None], []

    def run(r):
        try:
            st = ctxs[r].sweep()
            res[r] = (st, ctxs[r].extract(want_z=False)[0])
        except Exception as e:  # noqa: BLE001 -- reported below
            errs.append(repr(e))

    th = [threading.Thread(target=run, args=(r,)) for r in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=1200)
    for c in ctxs:
        c.close()
    assert not errs, errs
    for st, lam in res:
        assert st["converged"] and st["sweeps"] == _C3_LAM["bo"][1]
        assert np.array_equal(lam, _C3_LAM["bo"][0])


def test_c2_full_factor_reduce_sweep_vs_oracle(gh):
    """BASELINE configs[2]: LAPW 1568 x 1024 -> Phase 2 -> 1024^2 -> BO sweep, against the
    stored oracle reference of the same atoms (tests/golden/c2_oracle_bo: oracle.factor ->
    oracle BO on the tall Phase-1 factors, no Phase 2 -- Phase 2 preserves the pencil,
    eq 5.1, so its eigenvalues are the reference for any reduction); the device's Phase 2
    preserves the Grammians."""
    kind, at = inputs.make_config(2)
    NA, NL, NG = at.A.shape
    m = 2 * NA * NL
    meta = json.load(open(os.path.join(GOLD, "c2_oracle_bo.json")))
    lo = np.load(os.path.join(GOLD, "c2_oracle_bo.npz"))["lam"]
    assert inputs.fingerprint_close(inputs.fingerprint(at), meta["fingerprint"])
    ctx = gh.Context(m, NG, NL, variant="bo")
    ctx.factor(at.A, at.B, at.U, at.TAA, at.TAB, at.TBB)
    Ft, Jt, Gt, _ = ctx.get_factors()
    ctx.reduce()
    Fr, Jr, Gr, p2 = ctx.get_factors()
    assert Fr.shape == (NG, NG)
    Ht = Ft.conj().T @ (Jt[:, None] * Ft)
    St = Gt.conj().T @ Gt
    assert np.linalg.norm(Fr.conj().T @ (Jr[:, None] * Fr) - Ht[np.ix_(p2, p2)]) / np.linalg.norm(Ht) < 1e-10
    assert np.linalg.norm(Gr.conj().T @ Gr - St[np.ix_(p2, p2)]) / np.linalg.norm(St) < 1e-11
    st = ctx.sweep()
    lam, sf, sg, Z = ctx.extract()
    ctx.close()
    err = float(np.max(np.abs(np.sort(lam) - np.sort(lo)) / np.abs(np.sort(lo))))
    print(f"c2 reduced GPU vs tall oracle: max rel lambda err {err:.2e}, sweeps {st['sweeps']} "
          f"(oracle tall {meta['stats']['sweeps']})")
    assert st["converged"] and meta["stats"]["converged"]
    # Phase 2's hyperbolic (J-orthogonal, not unitary) reflectors preserve the Grammians
    # only to ~2e-12 relative (measured), which moves the eigenvalues by ~1e-9 relative
    # whichever implementation reduces (the oracle's own Phase 2 differs from the device's
    # by 3.8e-9, the blocked device path by 1.5e-9): bound 1e-8 here; the sweep itself is
    # held to 1e-9 on the tall factors below.
    assert err <= 1e-8
    ctx2 = gh.Context(m, NG, NL, variant="bo")
    ctx2.factor(at.A, at.B, at.U, at.TAA, at.TAB, at.TBB)
    st2 = ctx2.sweep()
    lam2 = ctx2.extract(want_z=False)[0]
    ctx2.close()
    err2 = float(np.max(np.abs(np.sort(lam2) - np.sort(lo)) / np.abs(np.sort(lo))))
    print(f"c2 tall GPU vs tall oracle: max rel lambda err {err2:.2e}, sweeps {st2['sweeps']}")
    assert st2["converged"] and err2 <= 1e-9 and abs(st2["sweeps"] - meta["stats"]["sweeps"]) <= 1
    # eigenvectors of the ORIGINAL (Phase-1) pencil through P2 un-permutation
    idx = np.arange(0, NG, 37)
    x = Z[:, idx]
    nf2 = np.linalg.norm(Ft) ** 2 + np.linalg.norm(Gt) ** 2
    r = np.linalg.norm(Ht @ x - (St @ x) * lam[idx][None, :], axis=0) / (nf2 * np.linalg.norm(x, axis=0))
    assert r.max() <= 1e-12 * NG


def test_c3_converged_lambda_vs_stored_oracle(gh, c3):
    """The headline config's converged eigenvalues against the oracle's (pointwise Alg. 2 on
    the oracle's own Phase-1 factors of the same atoms): <= 1e-6 per eigenvalue (north
    star, ill-conditioned).  BO from the bench-configuration solve above, pointwise solved
    here; sweep counts: pointwise within +-1 of the oracle's pointwise count."""
    meta, lo = _stored_c3("pointwise")
    assert inputs.fingerprint_close(inputs.fingerprint(c3), meta["fingerprint"]), \
        "config-3 inputs differ from those the stored oracle reference was computed on"
    assert meta["stats"]["converged"]
    if "bo" not in _C3_LAM:
        pytest.fail("needs the BO solve of test_c3_blocked_converges_with_residuals")
    err_bo = _relerr(_C3_LAM["bo"][0], lo)
    ctx = _ctx_c3(gh, c3, variant="pointwise", max_sweeps=64)
    st = ctx.sweep()
    lam = ctx.extract(want_z=False)[0].copy()
    ctx.close()
    err_pw = _relerr(lam, lo)
    print(f"c3 vs stored oracle (pointwise, {meta['stats']['sweeps']} sweeps): BO err {err_bo:.2e} "
          f"({_C3_LAM['bo'][1]} sweeps), pointwise err {err_pw:.2e} ({st['sweeps']} sweeps)")
    assert err_bo <= 1e-6 and err_pw <= 1e-6
    assert st["converged"] and abs(st["sweeps"] - meta["stats"]["sweeps"]) <= 1
    bo = os.path.join(GOLD, "c3_oracle_bo.json")
    if os.path.exists(bo):
        mb, lb = _stored_c3("bo")
        assert _relerr(_C3_LAM["bo"][0], lb) <= 1e-6
        assert abs(_C3_LAM["bo"][1] - mb["stats"]["sweeps"]) <= 1


def test_c3_hier_ordering_converged_lambda_vs_stored_oracle(gh, c3):
    """The bench's configuration of the headline config: BO in the HIER block ordering
    (4 super blocks, reading R2-5) -- converged eigenvalues <= 1e-6 of the oracle's stored
    pointwise solve, residuals on sampled pairs as for the round-robin solve."""
    meta, lo = _stored_c3("pointwise")
    assert inputs.fingerprint_close(inputs.fingerprint(c3), meta["fingerprint"])
    ctx = _ctx_c3(gh, c3, variant="bo", max_sweeps=64, ordering="hier", super_blocks=4)
    st = ctx.sweep()
    lam = ctx.extract(want_z=False)[0].copy()
    ctx.close()
    err = _relerr(lam, lo)
    print(f"c3 HIER: {st['sweeps']} sweeps, {st['seconds']:.2f} s, lambda vs stored oracle {err:.2e}")
    assert st["converged"] and err <= 1e-6


@pytest.fixture(scope="module")
def c4():
    kind, at = inputs.make_config(4)
    return at


def test_c4_first_block_step_matches_oracle(gh, c4):
    """BASELINE configs[4] at full size (30976 x 8192): the oracle's own Phase-1 factors go
    to the device (set_factors); after block step 0 of the bench's launch configuration
    (BO, auto partition 256 x w = 32) every 16th block pair's F, G, Z columns match
    oracle.block_pair run on the same columns (Sec 6.4.2-6.4.3)."""
    import torch
    at = c4
    F, J, G = oracle.factor(at.A, at.B, at.U, at.TAA, at.TAB, at.TBB)
    m, n = F.shape
    ctx = gh.Context(m, n, variant="bo")
    ctx.set_factors(F, J, G)
    ctx.run_steps(0, 1)
    dev = "cuda"
    Ft = torch.empty((n, m), dtype=torch.complex128, device=dev)    # column-major m x n
    Gt = torch.empty((n, m), dtype=torch.complex128, device=dev)
    Zt = torch.empty((n, n), dtype=torch.complex128, device=dev)
    import ctypes
    rc = ctx._L.ghsvd_get_transformed(ctx._h, ctypes.c_void_p(Ft.data_ptr()), m, ctypes.c_void_p(Gt.data_ptr()),
                                      m, ctypes.c_void_p(Zt.data_ptr()), n)
    ctx._check(rc, "get_transformed")
    torch.cuda.synchronize()
    ctx.close()
    perm = np.argsort(-J, kind="stable")       # device rows of F are J-sorted (+ first), stably; G's as given
    nblk = 2 * ((n + 63) // 64)
    start, width = oracle.block_partition(n, nblk)
    worst = 0.0
    for k in range(0, nblk // 2, 16):
        p, q = oracle.rr_pair(nblk, 0, k)
        cols = np.r_[start[p]:start[p] + width[p], start[q]:start[q] + width[q]]
        Fp = np.asfortranarray(F[:, cols])
        Gp = np.asfortranarray(G[:, cols])
        Zp = np.asfortranarray(np.eye(len(cols), dtype=complex))
        oracle.block_pair(Fp, J, Gp, Zp, 0, width[p], width[p], width[q])
        ci = torch.from_numpy(cols).to(dev)
        Fg = Ft.index_select(0, ci).T.cpu().numpy()
        Gg = Gt.index_select(0, ci).T.cpu().numpy()
        Zg = Zt.index_select(0, ci).T.cpu().numpy()[cols]
        for X, Y in ((Fg, Fp[perm]), (Gg, Gp)):
            e = np.linalg.norm(X - Y, axis=0) / np.linalg.norm(Y, axis=0)
            worst = max(worst, float(e.max()))
        worst = max(worst, float((np.linalg.norm(Zg - Zp, axis=0) / np.linalg.norm(Zp, axis=0)).max()))
    print(f"c4 block step 0: max rel column error {worst:.2e}")
    # same reasoning and bound as the config-3 block step above
    assert worst < 1e-8


def test_c4_blocked_converges_with_residuals(gh, c4):
    """Config 4 end to end (Phase 1 on the device, BO to convergence): sampled residuals, and
    the converged eigenvalues against the stored dense oracle reference of the same atoms
    (tests/golden/c4_oracle_dense.*: oracle.factor -> oracle.pencil_eigvals, the paper's
    form-H-and-S route, exact to ~eps kappa(S) with kappa(S) ~ 10 here)
    at the north-star well-conditioned tolerance 1e-9 per eigenvalue."""
    at = c4
    NA, NL, NG = at.A.shape
    ctx = gh.Context(2 * NA * NL, NG, NL, variant="bo", max_sweeps=64)
    ctx.factor(at.A, at.B, at.U, at.TAA, at.TAB, at.TBB)
    F0, J0, G0, _ = ctx.get_factors()
    st = ctx.sweep()
    lam, sf, sg, Z = ctx.extract()
    ctx.close()
    print("c4", st["sweeps"], st["kernel_seconds"])
    assert st["converged"]
    stem = os.path.join(GOLD, "c4_oracle_dense")
    if not os.path.exists(stem + ".json"):
        pytest.fail(f"missing stored oracle reference {stem}.json (tools/make_oracle_reference.py)")
    meta = json.load(open(stem + ".json"))
    assert inputs.fingerprint_close(inputs.fingerprint(at), meta["fingerprint"]), \
        "config-4 inputs differ from those the stored oracle reference was computed on"
    err = _relerr(lam, np.load(stem + ".npz")["lam"])
    print(f"c4 lambda vs stored dense oracle: {err:.2e} (kappa(S) {meta['stats']['kappa_S']:.3g})")
    assert err <= 1e-9
    idx = np.random.default_rng(1).choice(NG, 24, replace=False)
    x = Z[:, idx]
    nf2 = np.linalg.norm(F0) ** 2 + np.linalg.norm(G0) ** 2
    Hx = F0.conj().T @ (J0[:, None] * (F0 @ x))
    Sx = G0.conj().T @ (G0 @ x)
    res = np.linalg.norm(Hx - Sx * lam[idx][None, :], axis=0) / (nf2 * np.linalg.norm(x, axis=0))
    assert res.max() <= 1e-12 * NG


@pytest.mark.parametrize("ordering", ["hier", "rr"])
def test_c5_converged_lambda_vs_stored_oracle(gh, ordering):
    """Dataset C at n = 4000 (config 5, the paper's GSVD workload; J = I):
    BO in the bench's HIER ordering and in the round-robin against the stored oracle solve
    of the same seeded pencil (tests/golden/c5_oracle_pointwise.*, oracle.hz_pointwise to
    convergence on the pencil as generated), per eigenvalue."""
    stem = os.path.join(GOLD, "c5_oracle_pointwise")
    if not os.path.exists(stem + ".json"):
        pytest.fail(f"missing stored oracle reference {stem}.json (tools/make_oracle_reference.py)")
    meta = json.load(open(stem + ".json"))
    kind, P = inputs.make_config(5)
    assert inputs.fingerprint_close(inputs.fingerprint(P), meta["fingerprint"])
    n = P.F.shape[1]
    kw = dict(ordering="hier", super_blocks=4) if ordering == "hier" else {}
    ctx = gh.Context(n, n, variant="bo", max_sweeps=64, **kw)
    ctx.set_factors(P.F, P.J, P.G)
    st = ctx.sweep()
    lam = ctx.extract(want_z=False)[0].copy()
    ctx.close()
    err = _relerr(lam, np.load(stem + ".npz")["lam"])
    print(f"c5 {ordering}: {st['sweeps']} sweeps (oracle {meta['stats']['sweeps']}), lambda vs stored oracle {err:.2e}")
    assert st["converged"] and err <= C5_TOL
