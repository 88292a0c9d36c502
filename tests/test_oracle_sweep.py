"""Pins for the oracle's whole-sweep algorithms (no GPU).

Pinned to: closed-form spectra of pencils built with known generalized
singular values (BASELINE north_star; SURVEY C-20, C-21), the S = I special
case reducing to a Hermitian eigenproblem (numpy eigvalsh), a Cholesky-free
brute force in mpmath at 40 digits on tiny general pencils, the GHSVD
definition (V^*V = I, F columns J-orthogonal,
Sigma_F^2 + Sigma_G^2 = 1), the congruence F_c = F Z', and residuals.
"""
import os

import numpy as np
import pytest

import oracle
from paper_1907_08560_b200 import inputs

EPS = oracle.EPS


def relerr(a, b):
    a = np.sort(np.asarray(a))
    b = np.sort(np.asarray(b))
    return float(np.max(np.abs(a - b) / np.abs(b)))


def residual(F, J, G, lam, Z):
    """BASELINE residual ||Hx - lam Sx|| / ((||F||_F^2 + ||G||_F^2) ||x||), per column (C-15)."""
    nf2 = np.linalg.norm(F) ** 2 + np.linalg.norm(G) ** 2
    Hx = F.conj().T @ (J[:, None] * (F @ Z))
    Sx = G.conj().T @ (G @ Z)
    r = np.linalg.norm(Hx - Sx * lam[None, :], axis=0) / (nf2 * np.linalg.norm(Z, axis=0))
    return float(r.max())


def run(P, **kw):
    F, G, Zp, st = oracle.hz_pointwise(P.F, P.J, P.G, **kw)
    lam, sf, sg, Z = oracle.extract(F, P.J, G, Zp)
    return F, G, Zp, st, lam, sf, sg, Z


@pytest.mark.parametrize("m,n,seed", [(64, 32, 1), (128, 64, 2), (96, 96, 3), (200, 40, 4)])
def test_known_gsvd_J_identity(m, n, seed):
    """J = I: lambda = alpha^2/beta^2 exactly (config-1 recipe, BASELINE configs[1])."""
    P = inputs.known_gsvd(seed, m, n)
    F, G, Zp, st, lam, sf, sg, Z = run(P)
    assert st["converged"] and st["big_per_sweep"][-1] == 0
    assert relerr(lam, P.lam_true) < 1e-10
    assert residual(P.F, P.J, P.G, lam, Z) < 1e-12 * n
    # GHSVD definition: Sigma_F^2 + Sigma_G^2 = 1 ; V = G' Sigma_G'^-1 unitary
    assert np.allclose(sf ** 2 + sg ** 2, 1.0, atol=4 * EPS)
    V = G / np.linalg.norm(G, axis=0)
    assert np.abs(V.conj().T @ V - np.eye(n)).max() < 1e-12
    # congruence: converged factors equal the inputs times the accumulated Z'
    assert np.linalg.norm(F - P.F @ Zp) / np.linalg.norm(F) < 1e-11
    assert np.linalg.norm(G - P.G @ Zp) / np.linalg.norm(G) < 1e-11
    # at convergence no pair passes the relative criterion (C-1/C-3, J = I)
    tol = EPS * np.sqrt(n)
    Hm = F.conj().T @ F
    Sm = G.conj().T @ G
    d = 1 / np.sqrt(np.diag(Sm).real)
    Hs = Hm * np.outer(d, d)
    Ss = Sm * np.outer(d, d)
    off = np.abs(Hs) / np.sqrt(np.outer(np.abs(np.diag(Hs)), np.abs(np.diag(Hs))))
    np.fill_diagonal(off, 0)
    so = np.abs(Ss - np.diag(np.diag(Ss)))
    assert off.max() < 1e3 * tol and so.max() < 1e3 * tol


@pytest.mark.parametrize("m,n,seed,neg", [(64, 32, 5, 0.4), (128, 64, 6, 0.5), (80, 80, 7, 0.3), (160, 48, 8, 0.6)])
def test_known_hyperbolic(m, n, seed, neg):
    """J != I: lambda_i = j'_i alpha_i^2 / beta_i^2 with Q_J J-unitary (C-21)."""
    P = inputs.known_hyperbolic(seed, m, n, neg)
    F, G, Zp, st, lam, sf, sg, Z = run(P)
    assert st["converged"]
    assert relerr(lam, P.lam_true) < 1e-10
    assert residual(P.F, P.J, P.G, lam, Z) < 1e-12 * n
    # converged F columns mutually J-orthogonal
    Hc = F.conj().T @ (P.J[:, None] * F)
    nrm = np.sqrt(np.abs(np.diag(Hc)))
    off = np.abs(Hc) / np.outer(nrm, nrm)
    np.fill_diagonal(off, 0)
    assert off.max() < 1e-10
    assert np.all(np.sign(lam) == np.sign(np.diag(Hc).real))


@pytest.mark.parametrize("seed", [11, 12])
def test_orthonormal_G_reduces_to_hermitian_eig(seed):
    """S = I special case: lambda = eig(F^* J F) by an independent library routine."""
    P = inputs.orthonormal_G(seed, 90, 40)
    _, _, _, st, lam, *_ = run(P)
    H = P.F.conj().T @ (P.J[:, None] * P.F)
    ref = np.linalg.eigvalsh(0.5 * (H + H.conj().T))
    assert relerr(lam, ref) < 1e-10


def _mp_brute(F, J, G, dps=40):
    """Cholesky-free brute force at dps digits: S = Q L Q^*, S^{-1/2} H S^{-1/2} eigenvalues."""
    import mpmath as mp
    mp.mp.dps = dps
    n = F.shape[1]
    Fm = mp.matrix(F.tolist())
    Gm = mp.matrix(G.tolist())
    Jm = mp.diag([int(j) for j in J])
    H = Fm.H * Jm * Fm
    S = Gm.H * Gm
    ev, Q = mp.eighe(S)
    Sih = Q * mp.diag([1 / mp.sqrt(e) for e in ev]) * Q.H
    A = Sih * H * Sih
    A = (A + A.H) / 2
    w, _ = mp.eighe(A)
    return np.array([float(w[i]) for i in range(n)])


@pytest.mark.parametrize("m,n,seed", [(10, 6, 21), (16, 12, 22), (20, 9, 23)])
def test_mpmath_bruteforce_tiny(m, n, seed):
    """Tiny general pencils (odd n exercises bordering, Sec 6.3.2) vs 40-digit brute force."""
    P = inputs.random_pencil(seed, m, n, 0.5)
    _, _, _, st, lam, *_ = run(P)
    ref = _mp_brute(P.F, P.J, P.G)
    assert relerr(lam, ref) < 1e-11


def test_illconditioned_small_analog_vs_mpmath():
    """Config-3 analog (coupled, S singular values 1 ... 1e-12, C-14) vs 60-digit brute force:
    the GHSVD keeps eigenvalue accuracy where Cholesky-based solvers lose ~1e-6."""
    at = inputs.illcond_atoms(31, 2, 5, 12, smin=1e-6)
    F, J, G = oracle.factor(at.A, at.B, at.U, at.TAA, at.TAB, at.TBB)
    Fo, Go, Zp, st = oracle.hz_pointwise(F, J, G)
    lam, *_ = oracle.extract(Fo, J, Go, Zp)
    ref = _mp_brute(F, J, G, dps=60)
    assert relerr(lam, ref) < 1e-8


def test_determinism_across_threads():
    """PAPER.md:529-535 reproducibility: same inputs -> bitwise same outputs for any thread count."""
    P = inputs.known_hyperbolic(9, 96, 64, 0.5)
    a = oracle.hz_pointwise(P.F, P.J, P.G, nthreads=1)
    b = oracle.hz_pointwise(P.F, P.J, P.G, nthreads=4)
    for x, y in zip(a[:3], b[:3]):
        assert np.array_equal(x, y)
    assert a[3] == b[3]


def test_steps_equal_first_sweep():
    """or_hz_steps over all n-1 steps == the first sweep of Algorithm 2 (bitwise)."""
    P = inputs.random_pencil(10, 40, 20, 0.5)
    n = 20
    F1, G1, Z1, st = oracle.hz_pointwise(P.F, P.J, P.G, cmax=1)
    Z0 = np.eye(n, dtype=complex)
    F2, G2, Z2, a, b = oracle.hz_steps(P.F, P.J, P.G, Z0, 0, n - 1)
    F3, G3, Z3, a1, b1 = oracle.hz_steps(P.F, P.J, P.G, Z0, 0, 7)
    F3, G3, Z3, a2, b2 = oracle.hz_steps(F3, P.J, G3, Z3, 7, n - 8)
    assert np.array_equal(F1, F2) and np.array_equal(G1, G2) and np.array_equal(Z1, Z2)
    assert np.array_equal(F2, F3) and np.array_equal(Z2, Z3)
    assert st["transforms_all"] == a == a1 + a2 and st["transforms_big"] == b == b1 + b2


def test_stop_rule_and_cmax():
    """C-3: stop when a sweep has no big transform; C_max caps the sweeps (not converged)."""
    P = inputs.known_gsvd(3, 64, 32)
    *_, st, lam, sf, sg, Z = run(P, cmax=3)
    assert st["sweeps"] == 3 and not st["converged"]
    *_, st, lam, sf, sg, Z = run(P, cmax=30)
    assert st["converged"] and st["big_per_sweep"][-1] == 0 and all(b > 0 for b in st["big_per_sweep"][:-1])


def test_literal_criterion_same_eigenvalues():
    """C-1: the literal (6.12) reading gives the same lambda when stopping on big == 0."""
    P = inputs.known_hyperbolic(13, 64, 32, 0.5)
    *_, st1, l1, _, _, _ = run(P, criterion=oracle.CRIT_RELATIVE)
    *_, st2, l2, _, _, _ = run(P, criterion=oracle.CRIT_LITERAL)
    assert relerr(l1, P.lam_true) < 1e-10 and relerr(l2, P.lam_true) < 1e-10


@pytest.mark.parametrize("nblk,inner", [(4, 1), (8, 1), (6, 1), (10, 1), (8, 30)])
def test_blocked_matches_known_spectrum(nblk, inner):
    """Level-2 BO (inner 1 sweep) and FB (inner to convergence), Sec 6.4: same lambda;
    nblk = 6, 10 with n = 64 give widths w, w-1 and odd block pivots (bordered)."""
    P = inputs.known_hyperbolic(14, 96, 64, 0.4)
    F, G, Zp, st = oracle.hz_blocked(P.F, P.J, P.G, nblk, inner_sweeps=inner)
    lam, sf, sg, Z = oracle.extract(F, P.J, G, Zp)
    assert st["converged"]
    assert relerr(lam, P.lam_true) < 1e-10
    assert residual(P.F, P.J, P.G, lam, Z) < 1e-12 * 64


# -------------------------------------------------------------- HEBPJ / pchol
@pytest.mark.parametrize("r,seed", [(1, 0), (2, 1), (7, 2), (8, 3), (40, 4), (98, 5), (162, 6)])
def test_hebpj_reconstruction_and_inertia(r, seed):
    """Sec 4.2-4.3: T = M^* J M, J sorted (+ first); #(+) equals the number of positive
    eigenvalues (Sylvester's law of inertia, numpy eigvalsh)."""
    rng = np.random.default_rng(seed)
    X = inputs.cgauss(rng, (r, r))
    T = X + X.conj().T
    M, J, npos = oracle.hebpj(T)
    assert np.linalg.norm(M.conj().T @ (J[:, None] * M) - T) / np.linalg.norm(T) < 100 * r * r * EPS
    assert npos == int((np.linalg.eigvalsh(T) > 0).sum())
    assert np.all(J[:npos] == 1) and np.all(J[npos:] == -1)


def test_hebpj_golden():
    import json, os
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))["hebpj"]
    for ex in g:
        T = np.array([[complex(*v) for v in row] for row in ex["T"]])
        M, J, npos = oracle.hebpj(T)
        assert list(J) == ex["J"], ex["cite"]
        if "absM" in ex:
            assert np.allclose(np.abs(M), ex["absM"], atol=4 * EPS), ex["cite"]
        assert np.allclose(M.conj().T @ (J[:, None] * M), T, atol=8 * EPS)


def test_hebpj_rank_deficient_raises():
    T = np.zeros((3, 3), complex)
    with pytest.raises(oracle.OracleError):
        oracle.hebpj(T)


def test_pchol():
    rng = np.random.default_rng(7)
    for r in (1, 5, 33):
        X = inputs.cgauss(rng, (r + 3, r))
        S = X.conj().T @ X
        Gh = oracle.pchol(S)
        assert np.linalg.norm(Gh.conj().T @ Gh - S) / np.linalg.norm(S) < 50 * r * EPS
    with pytest.raises(oracle.OracleError):
        oracle.pchol(-np.eye(2, dtype=complex))


# ------------------------------------------------------------- phases 1, 2
def _HS_from_atoms(at):
    NA = at.A.shape[0]
    H = 0
    S = 0
    for a in range(NA):
        T = np.block([[at.TAA[a], at.TAB[a]], [at.TAB[a].conj().T, at.TBB[a]]])
        Ha = np.vstack([at.A[a], at.B[a]])
        Sa = np.vstack([at.A[a], at.U[a][:, None] * at.B[a]])
        H = H + Ha.conj().T @ T @ Ha                    # eq (4.1)
        S = S + Sa.conj().T @ Sa
    return H, S


@pytest.mark.parametrize("NA,NL,NG,neg", [(2, 4, 12, 0.5), (3, 5, 20, 0.4), (4, 9, 40, 0.5)])
def test_factor_grammians(NA, NL, NG, neg):
    """Phase 1 (Alg. 1, eqs 4.1-4.2): F^* J F = sum_a H_a^* T_a H_a, G^* G = sum_a S_a^* S_a;
    per-atom #(-) = number of negative eigenvalues of T_a (inertia)."""
    at = inputs.lapw_atoms(40 + NA, NA, NL, NG, neg)
    F, J, G = oracle.factor(at.A, at.B, at.U, at.TAA, at.TAB, at.TBB)
    H, S = _HS_from_atoms(at)
    assert np.linalg.norm(F.conj().T @ (J[:, None] * F) - H) / np.linalg.norm(H) < 1e-13
    assert np.linalg.norm(G.conj().T @ G - S) / np.linalg.norm(S) < 1e-14
    for a in range(NA):
        blk = J[2 * NL * a: 2 * NL * (a + 1)]
        assert (blk < 0).sum() == (at.d[a] < 0).sum()
        assert np.all(np.diff(blk.astype(int)) <= 0)   # + before -


@pytest.mark.parametrize("m,n,neg", [(60, 12, 0.5), (200, 40, 0.4), (150, 150, 0.5), (300, 64, 0.1)])
def test_reduce_grammian_preservation(m, n, neg):
    """Phase 2 (eq 5.1): P2^T Ft^* Jt Ft P2 = F^* J F, likewise for G; F block upper
    triangular (1x1/2x2 diagonal blocks), G upper triangular with real diagonal >= 0."""
    P = inputs.random_pencil(50 + m, m, n, neg)
    Fs, Js, Gs, p2, n2 = oracle.reduce(P.F, P.J, P.G)
    H = P.F.conj().T @ (P.J[:, None] * P.F)
    S = P.G.conj().T @ P.G
    assert sorted(p2) == list(range(n))
    Hp = H[np.ix_(p2, p2)]
    Sp = S[np.ix_(p2, p2)]
    assert np.linalg.norm(Fs.conj().T @ (Js[:, None] * Fs) - Hp) / np.linalg.norm(H) < 1e-11
    assert np.linalg.norm(Gs.conj().T @ Gs - Sp) / np.linalg.norm(S) < 1e-12
    assert np.abs(np.tril(Fs, -2)).max() == 0 and np.abs(np.tril(Gs, -1)).max() == 0
    assert np.all(np.diag(Gs).real >= 0) and np.all(np.diag(Gs).imag == 0)


def test_reduce_then_sweep_same_eigenvalues():
    """the GHSVD is invariant under Phase 2 (Lambda unchanged)."""
    at = inputs.lapw_atoms(60, 4, 6, 30, 0.4)
    F, J, G = oracle.factor(at.A, at.B, at.U, at.TAA, at.TAB, at.TBB)
    Fo, Go, Zp, _ = oracle.hz_pointwise(F, J, G)
    l1, *_ = oracle.extract(Fo, J, Go, Zp)
    Fs, Js, Gs, p2, n2 = oracle.reduce(F, J, G)
    Fo, Go, Zp, _ = oracle.hz_pointwise(Fs, Js, Gs)
    l2, *_ = oracle.extract(Fo, Js, Go, Zp)
    assert relerr(l2, l1) < 1e-9


# -------------------------------------------------------------- block pivots
@pytest.mark.parametrize("n,nblk", [(64, 8), (64, 6), (67, 10), (33, 2), (100, 16)])
def test_block_partition_definition(n, nblk):
    """Sec 6.4.1: exactly nblk block columns of widths w or w-1
    (w = ceil(n/nblk)), non-increasing, covering 0..n-1 contiguously."""
    start, width = oracle.block_partition(n, nblk)
    w = -(-n // nblk)
    assert len(width) == nblk and width.sum() == n
    assert set(width.tolist()) <= {w, w - 1} and all(np.diff(width) <= 0)
    assert start[0] == 0 and np.array_equal(start[1:], np.cumsum(width)[:-1])


def test_block_pair_fb_diagonalises_and_is_a_congruence():
    """Sec 6.4.2-6.4.3: with the inner level iterated to convergence (FB) the pair's block
    columns become mutually J-orthogonal / orthogonal, the other columns are untouched, and
    the update is the congruence F_pair <- F_pair Z_blk accumulated into Z."""
    P = inputs.known_hyperbolic(71, 80, 24, 0.5)
    F = np.asfortranarray(P.F.copy())
    G = np.asfortranarray(P.G.copy())
    Z = np.asfortranarray(np.eye(24, dtype=np.complex128))
    cols = list(range(4, 10)) + list(range(15, 20))          # blocks [4,10) and [15,20): order 11 (bordered)
    a, b = oracle.block_pair(F, P.J, G, Z, 4, 6, 15, 5, inner_sweeps=30)
    assert a > 0
    Fp, Gp = F[:, cols], G[:, cols]
    H = Fp.conj().T @ (P.J[:, None] * Fp)
    S = Gp.conj().T @ Gp
    dh, ds = np.sqrt(np.abs(np.diag(H))), np.sqrt(np.diag(S).real)
    offH = np.abs(H) / np.outer(dh, dh)
    offS = np.abs(S) / np.outer(ds, ds)
    np.fill_diagonal(offH, 0)
    np.fill_diagonal(offS, 0)
    assert offH.max() < 1e-10 and offS.max() < 1e-12
    others = [c for c in range(24) if c not in cols]
    assert np.array_equal(F[:, others], P.F[:, others]) and np.array_equal(G[:, others], P.G[:, others])
    Zb = Z[np.ix_(cols, cols)]
    assert np.linalg.norm(F[:, cols] - P.F[:, cols] @ Zb) / np.linalg.norm(F[:, cols]) < 1e-12
    assert np.linalg.norm(G[:, cols] - P.G[:, cols] @ Zb) / np.linalg.norm(G[:, cols]) < 1e-12


# ------------------------------------------------ NEXT-1: accumulated Z'^{-1}
@pytest.mark.parametrize("which,m,n", [("hyp", 96, 64), ("gsvd", 128, 64), ("rand", 70, 40)])
def test_accumulated_inverse_and_eq71_errors(which, m, n):
    """W = Z'^{-1} accumulated by the 2x2 inverses from the left.
    Pins: W Z' = I (definition of the inverse, numpy matmul); the GHSVD (3.1) with
    X = Sigma W reproduces the inputs, i.e. the eq (7.1) relative errors
    ||F - U Sigma_F X||_F / ||F||_F and ||G - V Sigma_G X||_F / ||G||_F are at the level
    the paper reports (7.98e-14 ... 8.23e-13)."""
    if which == "hyp":
        P = inputs.known_hyperbolic(81, m, n, 0.5)
    elif which == "gsvd":
        P = inputs.known_gsvd(82, m, n)
    else:
        P = inputs.random_pencil(83, m, n, 0.5)
    F, G, Zp, W, st = oracle.hz_pointwise_inv(P.F, P.J, P.G)
    F2, G2, Zp2, st2 = oracle.hz_pointwise(P.F, P.J, P.G, nthreads=1)
    assert np.array_equal(F, F2) and np.array_equal(Zp, Zp2)      # same iteration
    assert np.abs(W @ Zp - np.eye(n)).max() < 1e-10
    lam, sf, sg, Z = oracle.extract(F, P.J, G, Zp)
    sfp = np.sqrt(np.abs(np.einsum("ij,i,ij->j", F.conj(), P.J, F).real))
    sgp = np.linalg.norm(G, axis=0)
    sig = np.sqrt(sfp ** 2 + sgp ** 2)
    U = F / sfp[None, :]
    V = G / sgp[None, :]
    X = sig[:, None] * W                                           # X = Sigma Z'^{-1}
    assert np.abs(Z @ X - np.eye(n)).max() < 1e-9                  # X = Z^{-1}
    eF = np.linalg.norm(P.F - U @ (sf[:, None] * X)) / np.linalg.norm(P.F)
    eG = np.linalg.norm(P.G - V @ (sg[:, None] * X)) / np.linalg.norm(P.G)
    assert eF < 1e-12 and eG < 1e-12


def test_datasetA_sign_structure_phase1():
    """Dataset A's sign structure: every J~_a has 3 positive and 239
    negative signs (N_L = 121); the oracle's HEBPJ reproduces that inertia per atom
    (Sylvester), sorted + first within each atom."""
    from paper_1907_08560_b200 import inputs
    at = inputs.lapw_atoms(60, 2, 121, 40, nneg=239)
    F, J, G = oracle.factor(at.A, at.B, at.U, at.TAA, at.TAB, at.TBB)
    for a in range(2):
        Ja = J[242 * a: 242 * (a + 1)]
        assert int((Ja > 0).sum()) == 3 and list(Ja[:3]) == [1, 1, 1]
        assert int((np.sign(at.d[a]) > 0).sum()) == 3


def test_stored_reference_script_and_fingerprint(tmp_path):
    """tools/make_oracle_reference.py (oracle only) writes lambda and the input fingerprint;
    the fingerprint accepts a regeneration of the same recipe and seed and rejects another
    seed (reading R2-2: stored references are keyed by their inputs)."""
    import json
    import subprocess
    import sys
    from paper_1907_08560_b200 import inputs
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "tools", "make_oracle_reference.py"), "--illcond",
                        "2,6,16,5", "--variant", "pointwise", "--threads", "2", "--out", str(tmp_path)],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    meta = json.load(open(tmp_path / "illcond_2_6_16_s5_oracle_pointwise.json"))
    lam = np.load(tmp_path / "illcond_2_6_16_s5_oracle_pointwise.npz")["lam"]
    assert meta["stats"]["converged"] and lam.shape == (16,) and meta["m"] == 24 and meta["n"] == 16
    assert inputs.fingerprint_close(inputs.fingerprint(inputs.illcond_atoms(5, 2, 6, 16)), meta["fingerprint"])
    assert not inputs.fingerprint_close(inputs.fingerprint(inputs.illcond_atoms(6, 2, 6, 16)), meta["fingerprint"])
    # the stored lambda is the oracle pipeline's own
    at = inputs.illcond_atoms(5, 2, 6, 16)
    F, J, G = oracle.factor(at.A, at.B, at.U, at.TAA, at.TAB, at.TBB)
    Fo, Go, Zp, st = oracle.hz_pointwise(F, J, G, cmax=64)
    assert np.array_equal(oracle.extract(Fo, J, Go, Zp)[0], lam)


def test_stored_dense_reference_script(tmp_path):
    """--variant dense (the config-4 reference: oracle.factor -> oracle.pencil_eigvals) writes
    the dense eigenvalues, kappa(S) and the input fingerprint, from the oracle alone."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "tools", "make_oracle_reference.py"), "--illcond",
                        "2,6,16,5", "--variant", "dense", "--threads", "2", "--out", str(tmp_path)],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    meta = json.load(open(tmp_path / "illcond_2_6_16_s5_oracle_dense.json"))
    lam = np.load(tmp_path / "illcond_2_6_16_s5_oracle_dense.npz")["lam"]
    at = inputs.illcond_atoms(5, 2, 6, 16)
    F, J, G = oracle.factor(at.A, at.B, at.U, at.TAA, at.TAB, at.TBB)
    assert np.array_equal(oracle.pencil_eigvals(F, J, G), lam)
    assert meta["stats"]["kappa_S"] >= 1.0 and meta["stats"]["negative"] == int((lam < 0).sum())
