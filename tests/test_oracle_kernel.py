"""Pins for the oracle's ordering and 2x2 transform (no GPU).

Each check is pinned to something other than the oracle itself: exhaustive
combinatorics (ordering), the defining invariants of the transform
(Z'^* S Z' = I and Z'^* H Z' diagonal, PAPER.md:1473-1482 and eq 6.8),
eigenvalues of the 2x2 pencil from numpy (an independent library routine),
hand-derived examples in tests/golden/spec_examples.json, and every branch
of Sec. 6.1.6 / 6.1.7 hit deliberately.
"""
import json
import os

import numpy as np
import pytest

import oracle

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))
EPS = oracle.EPS


def _c(v):
    return complex(v[0], v[1])


# ------------------------------------------------------------------ ordering
@pytest.mark.parametrize("n", list(range(2, 130, 2)) + [256, 512, 1024])
def test_round_robin_covers_every_pair_once(n):
    """a cyclic strategy has n-1 steps of n/2 disjoint pairs
    whose union is all n(n-1)/2 pairs; SURVEY C-11 round-robin."""
    seen = set()
    for s in range(n - 1):
        idx = set()
        for k in range(n // 2):
            p, q = oracle.rr_pair(n, s, k)
            assert 0 <= p < q < n
            assert p not in idx and q not in idx
            idx.update((p, q))
            assert (p, q) not in seen
            seen.add((p, q))
        assert len(idx) == n
    assert len(seen) == n * (n - 1) // 2


def test_round_robin_golden():
    g = GOLD["ordering"][0]
    n = g["n"]
    steps = [[oracle.rr_pair(n, s, k) for k in range(n // 2)] for s in range(n - 1)]
    assert len(steps) == g["steps"] and all(len(st) == g["pairs_per_step"] for st in steps)


def test_round_robin_rejects_bad_args():
    with pytest.raises(oracle.OracleError):
        oracle.rr_pair(5, 0, 0)
    with pytest.raises(oracle.OracleError):
        oracle.rr_pair(6, 5, 0)


# ----------------------------------------------------------------- 2x2 HZ
def _pivot(rng, kappa=None, jsig=(1, -1)):
    """Random Hermitian H (indefinite) and HPD S (optionally with condition kappa)."""
    A = rng.standard_normal((2, 2)) + 1j * rng.standard_normal((2, 2))
    if kappa is None:
        S = A.conj().T @ A
    else:
        Q, _ = np.linalg.qr(A)
        S = Q @ np.diag([1.0, 1.0 / kappa]) @ Q.conj().T
        S = S * rng.uniform(0.1, 10.0)
    B = rng.standard_normal((2, 2)) + 1j * rng.standard_normal((2, 2))
    H = B.conj().T @ np.diag(jsig) @ B
    H = 0.5 * (H + H.conj().T)
    S = 0.5 * (S + S.conj().T)
    return H, S


def _apply(H, S, n=64, criterion=oracle.CRIT_RELATIVE):
    return oracle.hz2x2(H[0, 0].real, H[1, 1].real, H[0, 1], S[0, 0].real, S[1, 1].real, S[0, 1], n,
                        criterion=criterion)


@pytest.mark.parametrize("kappa", [None, 1e1, 1e2, 1e4, 1e6])
def test_hz2x2_diagonalises_pencil(kappa):
    """eq (6.8) and PAPER.md:1473-1482: Z'^* S Z' = I, Z'^* H Z' diagonal; the
    diagonal equals the generalized eigenvalues of (H, S) (numpy eig), and
    Z' S-orthonormal.  Error bounds (measured): |Z'^*SZ' - I| <= c eps kappa(S),
    |offdiag Z'^*HZ'| <= c eps sqrt(kappa(S)) |H| |Z'|^2, c = 64."""
    rng = np.random.default_rng(11 if kappa is None else int(np.log10(kappa)) + 20)
    worst_s = worst_h = 0.0
    for _ in range(4000):
        H, S = _pivot(rng, kappa, jsig=tuple(rng.choice([-1, 1], 2)))
        kind, Z, off = _apply(H, S)
        assert kind in (oracle.K_SMALL, oracle.K_BIG)
        ZS = Z.conj().T @ S @ Z
        ZH = Z.conj().T @ H @ Z
        ks = np.linalg.cond(S)
        worst_s = max(worst_s, np.abs(ZS - np.eye(2)).max() / (EPS * ks))
        worst_h = max(worst_h, abs(ZH[0, 1]) / (EPS * np.sqrt(ks) * np.linalg.norm(H) * np.linalg.norm(Z) ** 2))
        lam = np.sort(np.linalg.eigvals(np.linalg.solve(S, H)).real)
        d = np.sort(ZH.diagonal().real / ZS.diagonal().real)
        assert np.allclose(d, lam, rtol=1e-8 * ks, atol=1e-10 * ks * np.abs(lam).max())
    assert worst_s < 64, worst_s
    assert worst_h < 64, worst_h


def test_hz2x2_golden_examples():
    for g in GOLD["hz2x2"]:
        H = np.array([[g["hpp"], _c(g["hpq"])], [np.conj(_c(g["hpq"])), g["hqq"]]])
        S = np.array([[g["spp"], _c(g["spq"])], [np.conj(_c(g["spq"])), g["sqq"]]])
        kind, Z, _ = oracle.hz2x2(g["hpp"], g["hqq"], _c(g["hpq"]), g["spp"], g["sqq"], _c(g["spq"]), g["n"])
        assert kind == g["kind"], g["cite"]
        if "diag_ZHZ" in g:
            ZH = Z.conj().T @ H @ Z
            ZS = Z.conj().T @ S @ Z
            assert np.allclose(sorted(ZH.diagonal().real), sorted(g["diag_ZHZ"]), atol=4 * EPS), g["cite"]
            assert np.allclose(ZS, np.diag(g["diag_ZSZ"]), atol=4 * EPS), g["cite"]
            assert abs(ZH[0, 1]) < 8 * EPS


def test_hz2x2_criterion_golden():
    for g in GOLD["criterion"]:
        n = g["n"]
        tol = EPS * np.sqrt(n)
        rc, _, _ = oracle.hz2x2_raw(g["hpp"], g["hqq"], g["hpq_scale"] * tol, 1.0, 1.0, g["spq_scale"] * tol, tol)
        assert (rc not in (oracle.K_SKIP,)) == g["transform"], g["cite"]


def test_hz2x2_x_zero_branch_is_plain_jacobi_rotation():
    """Sec 6.1.6 case 2: s_pq = 0 -> alpha_1 = 0, Z an ordinary (unitary) Jacobi rotation
    diagonalising H when S = I."""
    rng = np.random.default_rng(3)
    for _ in range(200):
        B = rng.standard_normal((2, 2)) + 1j * rng.standard_normal((2, 2))
        H = B + B.conj().T
        kind, Z, _ = _apply(H, np.eye(2))
        assert kind == oracle.K_BIG
        assert np.abs(Z.conj().T @ Z - np.eye(2)).max() < 8 * EPS
        ZH = Z.conj().T @ H @ Z
        assert abs(ZH[0, 1]) < 16 * EPS * np.linalg.norm(H)
        assert np.allclose(np.sort(ZH.diagonal().real), np.linalg.eigvalsh(H), atol=16 * EPS * np.linalg.norm(H))


def test_hz2x2_h_v_zero_branch():
    """Sec 6.1.6 case 3: h = v = 0 -> Z = R1 D2; check against the pencil invariants."""
    for x, a in [(0.0, 0.0), (0.3, 0.7), (0.9, -2.0), (0.999, 1.0)]:
        spq = x * np.exp(1j * a)
        for u in (0.5, -1.5):
            hpq = u * np.exp(1j * a)           # same argument as s_pq -> v = 0
            H = np.array([[2.0, hpq], [np.conj(hpq), 2.0]])
            S = np.array([[1.0, spq], [np.conj(spq), 1.0]])
            kind, Z, _ = _apply(H, S)
            assert kind == oracle.K_BIG
            assert np.abs(Z.conj().T @ S @ Z - np.eye(2)).max() < 64 * EPS / (1 - x)
            assert abs((Z.conj().T @ H @ Z)[0, 1]) < 64 * EPS / (1 - x)


def test_hz2x2_sigma_both_signs_and_scaling():
    """sigma = sgn(h) with both signs (C-4) and prescaling D0 (Sec 6.1.1): results
    scale covariantly when S's diagonal is scaled."""
    rng = np.random.default_rng(5)
    H, S = _pivot(rng)
    for hsign in (1.0, -1.0):
        Hs = H.copy()
        Hs[1, 1] = Hs[0, 0] + hsign * 0.25
        k1, Z1, _ = _apply(Hs, S)
        D = np.diag([3.0, 0.5])
        k2, Z2, _ = _apply(D @ Hs @ D, D @ S @ D)
        assert k1 == k2 == oracle.K_BIG
        # Z' for the scaled pencil equals D^{-1} Z' (same rotation after prescaling)
        assert np.allclose(D @ Z2, Z1, rtol=1e-13, atol=1e-13)


def test_hz2x2_small_and_skip_and_identity():
    n = 64
    tol = EPS * np.sqrt(n)
    # below the threshold -> skip
    rc, _, _ = oracle.hz2x2_raw(1.0, 2.0, 0.1 * tol, 1.0, 1.0, 0.0, tol)
    assert rc == oracle.K_SKIP
    # just above -> transformed, but tiny: cos(phi) = cos(psi) = 1 exactly -> small (C-2)
    rc, Z, _ = oracle.hz2x2_raw(1.0, 2.0, 4.0 * tol, 1.0, 1.0, 0.0, tol)
    assert rc == oracle.K_SMALL
    assert Z[0, 0] == 1.0 and Z[1, 1] == 1.0 and Z[0, 1] != 0
    # h_pq = s_pq = 0 with h_pp = 0 (relative threshold 0): identity, not counted
    rc, Z, _ = oracle.hz2x2_raw(0.0, 2.0, 0.0, 1.0, 1.0, 0.0, tol)
    assert rc == oracle.K_IDENTITY
    # literal criterion (eq 6.12 as printed) uses max*tol*min
    rc, _, _ = oracle.hz2x2_raw(1e-4, 1e-4, 1e-12, 1.0, 1.0, 0.0, tol, oracle.CRIT_LITERAL)
    assert rc != oracle.K_SKIP           # literal threshold ~ 1e-8*tol: transforms
    rc, _, _ = oracle.hz2x2_raw(1e-4, 1e-4, 1e-12, 1.0, 1.0, 0.0, tol, oracle.CRIT_RELATIVE)
    assert rc != oracle.K_SKIP           # relative threshold 1e-4*tol ~ 1e-19 : also transforms
    rc, _, _ = oracle.hz2x2_raw(1e-4, 1e-4, 1e-21, 1.0, 1.0, 0.0, tol, oracle.CRIT_RELATIVE)
    assert rc == oracle.K_SKIP


def test_hz2x2_errors():
    tol = EPS * 8
    assert oracle.hz2x2_raw(1.0, 1.0, 0.5, 0.0, 1.0, 0.1, tol)[0] == -6      # s_pp <= 0
    assert oracle.hz2x2_raw(1.0, 1.0, 0.5, 1.0, 1.0, 1.0, tol)[0] == -6      # x = 1: singular S (C-9)
    assert oracle.hz2x2_raw(np.nan, 1.0, 0.5, 1.0, 1.0, 0.1, tol)[0] == -8   # non-finite


# ------------------------------------------------------------------ J-dot golden
@pytest.mark.parametrize("case", GOLD["jdot"])
def test_jdot_golden_through_extract(case):
    """SPEC.md:55, 61 worked J-dots (f^* J f) pinned through the oracle's output formulas
    (reading C-16): with g = e_1, lambda = (f^* J f) / (g^* g) = f^* J f and
    Sigma'_F = |f^* J f|^(1/2).  The golden f equals g in both cases (a J-norm)."""
    f = np.array([_c(v) for v in case["f"]])
    J = np.array(case["J"], dtype=np.int8)
    want = _c(case["value"])
    F = np.zeros((2, 2), complex)
    G = np.zeros((2, 2), complex)
    F[:, 0], G[0, 0] = f, 1.0
    F[0, 1], G[1, 1] = 1.0, 1.0          # a second, orthogonal column (lambda = 1)
    lam, sf, sg, _ = oracle.extract(F, J, G, np.eye(2, dtype=complex))
    assert lam[0] == want.real and lam[1] == 1.0
    assert abs(sf[0] / sg[0] - np.sqrt(abs(want.real))) <= 4 * EPS * max(1.0, np.sqrt(abs(want.real)))
    assert sf[0] ** 2 + sg[0] ** 2 == pytest.approx(1.0, abs=4 * EPS)
