"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times.

Config 3 (10368 x 4096, S condition 1e12) is far beyond what the oracle can converge in a
test (the bench extrapolates ~80 min on 16 cores), so parity is checked
  * elementwise on the first step / block step against the oracle run on the same
    factors (ghsvd_get_factors), for sampled pairs, and
  * at convergence through properties that hold at any size: residual
    ||Hx - lambda Sx|| / ((||F||^2 + ||G||^2) ||x||) <= 1e-12 n for sampled eigenpairs
    (H, S never formed: Hx = F^*(J(Fx))), Sigma_F^2 + Sigma_G^2 = 1, G's columns
    orthonormal after normalisation.
Config 2 (LAPW 1568 x 1024 -> Phase 2 -> 1024^2) runs end to end against the oracle.
Config 4 (30976 x 8192) only with GHSVD_FULL=1 (minutes of GPU time).
"""
import os

import numpy as np
import pytest

import oracle
from paper_1907_08560_b200 import inputs

pytestmark = pytest.mark.gpu
EPS = oracle.EPS


@pytest.fixture(scope="module")
def gh():
    from paper_1907_08560_b200 import build, ghsvd
    build.build()
    return ghsvd


@pytest.fixture(scope="module")
def c3():
    kind, at = inputs.make_config(3, backend="torch")
    return at


_C3_LAM = {}   # eigenvalues of the bench-configuration solve, reused by later tests


def _ctx_c3(gh, at, **kw):
    NA, NL, NG = at.A.shape
    ctx = gh.Context(2 * NA * NL, NG, NL, **kw)
    ctx.factor(at.A, at.B, at.U, at.TAA, at.TAB, at.TBB)
    return ctx


def test_c3_pointwise_first_step_matches_oracle(gh, c3):
    ctx = _ctx_c3(gh, c3)
    F0, J0, G0, _ = ctx.get_factors()
    m, n = F0.shape
    a_g, b_g = ctx.run_steps(0, 1)
    Fg, Gg, Zg = ctx.transformed(m, n)
    ctx.close()
    Fo, Go, Zo, a, b = oracle.hz_steps(F0, J0, G0, np.eye(n, dtype=complex), 0, 1)
    assert (a_g, b_g) == (a, b)
    # Reduction order differs (tree vs sequential over m = 10368 rows) and the 2x2 transform
    # amplifies Gram perturbations by ~kappa of the pair's S block (S has condition 1e12 here):
    # 1e-10 relative per column (measured 2.5e-12).
    cols = np.r_[0:64, n - 64:n]
    for X, Y in ((Fg, Fo), (Gg, Go)):
        sc = np.linalg.norm(Y[:, cols], axis=0)
        assert (np.linalg.norm(X[:, cols] - Y[:, cols], axis=0) / sc).max() < 1e-10
    assert np.abs(Zg[:, cols] - Zo[:, cols]).max() < 1e-10


def test_c3_blocked_first_block_step_matches_oracle(gh, c3):
    ctx = _ctx_c3(gh, c3, variant="bo")
    F0, J0, G0, _ = ctx.get_factors()
    m, n = F0.shape
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
    for X, Y in ((Fg, F), (Gg, G)):
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
    """BASELINE configs[2]: LAPW 1568 x 1024 -> Phase 2 -> 1024^2 -> BO sweep, vs the oracle's
    blocked run (same partition) on the GPU's reduced factors; Phase 2 Grammians preserved."""
    kind, at = inputs.make_config(2)
    NA, NL, NG = at.A.shape
    m = 2 * NA * NL
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
    Fo, Go, Zp, sto = oracle.hz_blocked(Fr, Jr, Gr, 32, inner_sweeps=1)
    lo, *_ = oracle.extract(Fo, Jr, Go, Zp)
    assert st["converged"] and sto["converged"] and abs(st["sweeps"] - sto["sweeps"]) <= 1
    assert np.max(np.abs(np.sort(lam) - np.sort(lo)) / np.abs(np.sort(lo))) <= 1e-9
    # eigenvectors of the ORIGINAL (Phase-1) pencil through P2 un-permutation
    idx = np.arange(0, NG, 37)
    x = Z[:, idx]
    nf2 = np.linalg.norm(Ft) ** 2 + np.linalg.norm(Gt) ** 2
    r = np.linalg.norm(Ht @ x - (St @ x) * lam[idx][None, :], axis=0) / (nf2 * np.linalg.norm(x, axis=0))
    assert r.max() <= 1e-12 * NG


@pytest.mark.skipif(os.environ.get("GHSVD_FULL") != "1", reason="config 4 takes minutes; set GHSVD_FULL=1")
def test_c4_blocked_converges_with_residuals(gh):
    kind, at = inputs.make_config(4)
    NA, NL, NG = at.A.shape
    ctx = gh.Context(2 * NA * NL, NG, NL, variant="bo", max_sweeps=64)
    ctx.factor(at.A, at.B, at.U, at.TAA, at.TAB, at.TBB)
    F0, J0, G0, _ = ctx.get_factors()
    st = ctx.sweep()
    lam, sf, sg, Z = ctx.extract()
    ctx.close()
    print("c4", st["sweeps"], st["kernel_seconds"])
    assert st["converged"]
    idx = np.random.default_rng(1).choice(NG, 24, replace=False)
    x = Z[:, idx]
    nf2 = np.linalg.norm(F0) ** 2 + np.linalg.norm(G0) ** 2
    Hx = F0.conj().T @ (J0[:, None] * (F0 @ x))
    Sx = G0.conj().T @ (G0 @ x)
    res = np.linalg.norm(Hx - Sx * lam[idx][None, :], axis=0) / (nf2 * np.linalg.norm(x, axis=0))
    assert res.max() <= 1e-12 * NG
