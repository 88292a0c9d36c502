"""Pins for oracle.pencil_eigvals, the dense reference of the paper's "alternative way
forward" (form H = F^*JF and S = G^*G, solve with ZHEGVD; Sec 4.5), which
checks the GPU's converged eigenvalues on the well-conditioned full-size config 4.

Pinned to things other than itself: closed-form spectra of pencils built with known
generalized (hyperbolic) singular values (SURVEY C-20, C-21), the oracle's own HZ solve
(Alg. 2, an independent algorithm) on random pencils, the 2x2 closed form, and the sign
count of the spectrum (Sylvester's law of inertia: the pencil has as many negative
eigenvalues as H has, and H = F^*JF with F square nonsingular has inertia of J)."""
import numpy as np

import oracle
from paper_1907_08560_b200 import inputs


def relerr(a, b):
    a, b = np.sort(np.asarray(a)), np.sort(np.asarray(b))
    return float(np.max(np.abs(a - b) / np.abs(b)))


def test_known_hyperbolic_spectrum():
    P = inputs.known_hyperbolic(3, 160, 96, 0.4)
    assert relerr(oracle.pencil_eigvals(P.F, P.J, P.G), P.lam_true) <= 1e-10


def test_dense_loses_small_eigenvalues_when_S_is_ill_conditioned():
    """On the known-spectrum GSVD pencil (config 1's recipe: G = Q diag(beta) W with beta down
    to ~1e-2 and cond(W) = 1e3, so kappa(S) ~ 1e8) the dense route's smallest eigenvalue is off by
    more than 1e-10 while the implicit HZ keeps it to ~1e-13: the reason this reference
    is used for config 4 only."""
    P = inputs.known_gsvd(4, 200, 80)
    Fc, Gc, Zp, st = oracle.hz_pointwise(P.F, P.J, P.G)
    lam_hz, *_ = oracle.extract(Fc, P.J, Gc, Zp)
    e_dense = relerr(oracle.pencil_eigvals(P.F, P.J, P.G), P.lam_true)
    e_hz = relerr(lam_hz, P.lam_true)
    assert e_hz <= 1e-11 and e_dense > 10 * e_hz


def test_matches_hz_on_random_pencil():
    P = inputs.random_pencil(5, 120, 64, 0.5)
    Fc, Gc, Zp, st = oracle.hz_pointwise(P.F, P.J, P.G)
    lam_hz, *_ = oracle.extract(Fc, P.J, Gc, Zp)
    assert st["converged"]
    assert relerr(oracle.pencil_eigvals(P.F, P.J, P.G), lam_hz) <= 1e-10


def test_two_by_two_closed_form():
    # F = diag(a, b), J = diag(1, -1), G = I: H = diag(a^2, -b^2), S = I
    F = np.diag([3.0 + 0j, 2.0 + 0j])
    J = np.array([1, -1], dtype=np.int8)
    G = np.eye(2, dtype=complex)
    assert np.allclose(oracle.pencil_eigvals(F, J, G), [-4.0, 9.0], rtol=1e-15, atol=0)
    # G = diag(1, 2) scales the second eigenvalue by 1 / 4
    G = np.diag([1.0 + 0j, 2.0 + 0j])
    assert np.allclose(oracle.pencil_eigvals(F, J, G), [-1.0, 9.0], rtol=1e-15, atol=0)


def test_inertia_of_square_factor():
    rng = np.random.default_rng(6)
    n = 40
    F = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    G = rng.standard_normal((n + 8, n)) + 1j * rng.standard_normal((n + 8, n))
    J = np.where(rng.random(n) < 0.3, -1, 1).astype(np.int8)
    lam = oracle.pencil_eigvals(F, J, G)
    assert int((lam < 0).sum()) == int((J < 0).sum())


def test_matches_stored_hz_oracle_on_config2():
    """At a real LAPW shape: the dense route on the oracle's Phase-1 factors of config 2
    (1568 x 1024, well-conditioned S) against the stored HZ oracle solve of the same atoms
    (tests/golden/c2_oracle_bo.*, BO to convergence), per eigenvalue."""
    import json
    import os
    gold = os.path.join(os.path.dirname(__file__), "golden")
    meta = json.load(open(os.path.join(gold, "c2_oracle_bo.json")))
    lam_hz = np.load(os.path.join(gold, "c2_oracle_bo.npz"))["lam"]
    kind, at = inputs.make_config(2, backend="numpy")
    assert inputs.fingerprint_close(inputs.fingerprint(at), meta["fingerprint"])
    F, J, G = oracle.factor(at.A, at.B, at.U, at.TAA, at.TAB, at.TBB)
    assert relerr(oracle.pencil_eigvals(F, J, G), lam_hz) <= 1e-10
