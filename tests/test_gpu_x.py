"""NEXT-1 on the GPU: accumulating Z'^{-1} and X = Z^{-1} = Sigma Z'^{-1}.

Pins: X Z = I (definition of X in eq 3.2); the GHSVD (3.1) F = U Sigma_F X, G = V Sigma_G X
with the eq (7.1) relative errors at the paper's level (7.98e-14 ...
8.23e-13; bound 1e-12 here); W agrees with the oracle's accumulated inverse; the want_x
path leaves the eigenvalues bitwise unchanged (it only adds the W updates)."""
import numpy as np
import pytest

import oracle
from hostfactors import device_layout
from paper_1907_08560_b200 import inputs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gh():
    from paper_1907_08560_b200 import build, ghsvd
    build.build()
    return ghsvd


def eq71(F, J, G, Fc, Gc, X, sf, sg):
    """||F - U Sigma_F X||_F / ||F||_F and the G analogue, U = F' Sigma'_F^-1, V = G' Sigma'_G^-1."""
    sfp = np.sqrt(np.abs(np.einsum("ij,i,ij->j", Fc.conj(), J, Fc).real))
    sgp = np.linalg.norm(Gc, axis=0)
    U = Fc / sfp[None, :]
    V = Gc / sgp[None, :]
    eF = np.linalg.norm(F - U @ (sf[:, None] * X)) / np.linalg.norm(F)
    eG = np.linalg.norm(G - V @ (sg[:, None] * X)) / np.linalg.norm(G)
    return eF, eG


@pytest.mark.parametrize("variant,nb", [("pointwise", 0), ("bo", 4), ("bo", 6)])
def test_x_inverse_and_eq71(gh, variant, nb):
    P = inputs.known_hyperbolic(91, 160, 64, 0.5)
    m, n = P.F.shape
    runs = {}
    for wx in (False, True):
        ctx = gh.Context(m, n, variant=variant, nblocks=nb, want_x=wx)
        ctx.set_factors(P.F, P.J, P.G)
        F0, J0, G0 = device_layout(P.F, P.J, P.G)
        st = ctx.sweep()
        lam, sf, sg, Z = ctx.extract()
        X = ctx.extract_x() if wx else None
        Fc, Gc, Zp = ctx.transformed(m, n)
        ctx.close()
        runs[wx] = (F0, J0, G0, lam, sf, sg, Z, X, Fc, Gc, Zp, st)
    assert np.array_equal(runs[False][3], runs[True][3])          # eigenvalues untouched
    F0, J0, G0, lam, sf, sg, Z, X, Fc, Gc, Zp, st = runs[True]
    assert np.abs(Z @ X - np.eye(n)).max() < 1e-9
    eF, eG = eq71(F0, J0, G0, Fc, Gc, X, sf, sg)
    assert eF < 1e-12 and eG < 1e-12, (eF, eG)
    if variant == "pointwise":
        Fo, Go, Zo, Wo, sto = oracle.hz_pointwise_inv(F0, J0, G0)
        sig = np.sqrt(np.abs(np.einsum("ij,i,ij->j", Fo.conj(), J0, Fo).real) + np.linalg.norm(Go, axis=0) ** 2)
        Xo = sig[:, None] * Wo
        # two converged runs (different reduction orders) end on slightly different final
        # small rotations: eigenvector matrices agree to the convergence level, not to eps
        assert np.abs(X - Xo).max() / np.abs(Xo).max() < 1e-7


def test_x_after_phase2_is_in_original_column_order(gh):
    """With Phase 2 the columns of X~ = X P2^T refer to the Phase-1 factors."""
    at = inputs.lapw_atoms(92, 4, 10, 48, 0.4)
    ctx = gh.Context(80, 48, 10, want_x=True)
    ctx.factor(at.A, at.B, at.U, at.TAA, at.TAB, at.TBB)
    F1, J1, G1, _ = ctx.get_factors()
    ctx.reduce()
    ctx.sweep()
    lam, sf, sg, Z = ctx.extract()
    X = ctx.extract_x()
    ctx.close()
    assert np.abs(Z @ X - np.eye(48)).max() < 1e-9
    H = F1.conj().T @ (J1[:, None] * F1)
    S = G1.conj().T @ G1
    # X^* diag(Lambda_F) X = H and X^* diag(Lambda_G) X = S with Lambda_F = J Sigma_F^2
    LF = np.sign(lam) * sf ** 2
    LG = sg ** 2
    assert np.linalg.norm(X.conj().T @ (LF[:, None] * X) - H) / np.linalg.norm(H) < 1e-11
    assert np.linalg.norm(X.conj().T @ (LG[:, None] * X) - S) / np.linalg.norm(S) < 1e-11


def test_dataset_c_gsvd_small_vs_oracle(gh):
    """NEXT-3: dataset-C-like GSVD pair (J = I, Hermitian F, G with U(0,1) spectra,
    PAPER.md:2252-2257) at n = 128: eigenvalues vs the oracle, full GSVD residuals."""
    P = inputs.dataset_c(93, 128)
    ctx = gh.Context(128, 128, variant="bo", want_x=True)
    ctx.set_factors(P.F, P.J, P.G)
    F0, J0, G0 = device_layout(P.F, P.J, P.G)
    st = ctx.sweep()
    lam, sf, sg, Z = ctx.extract()
    X = ctx.extract_x()
    Fc, Gc, _ = ctx.transformed(128, 128)
    ctx.close()
    Fo, Go, Zp, sto = oracle.hz_pointwise(F0, J0, G0)
    lo, *_ = oracle.extract(Fo, J0, Go, Zp)
    assert st["converged"] and np.all(lam > 0)
    assert np.max(np.abs(np.sort(lam) - np.sort(lo)) / np.abs(np.sort(lo))) < 1e-9
    eF, eG = eq71(F0, J0, G0, Fc, Gc, X, sf, sg)
    assert eF < 1e-12 and eG < 1e-12


def test_x_with_cluster_pivot(gh, monkeypatch):
    """The two-CTA cluster block pivot (GHSVD_PIVOT_CL=1) with its separate Gauss-Jordan
    kernel for Z_blk^{-1}: X Z = I, eq 7.1 errors, eigenvalues bitwise unchanged by want_x."""
    monkeypatch.setenv("GHSVD_PIVOT_CL", "1")
    P = inputs.known_hyperbolic(92, 160, 64, 0.5)
    m, n = P.F.shape
    runs = {}
    for wx in (False, True):
        ctx = gh.Context(m, n, variant="bo", nblocks=6, want_x=wx)
        ctx.set_factors(P.F, P.J, P.G)
        F0, J0, G0 = device_layout(P.F, P.J, P.G)
        ctx.sweep()
        lam, sf, sg, Z = ctx.extract()
        X = ctx.extract_x() if wx else None
        Fc, Gc, Zp = ctx.transformed(m, n)
        ctx.close()
        runs[wx] = (F0, J0, G0, lam, sf, sg, Z, X, Fc, Gc)
    assert np.array_equal(runs[False][3], runs[True][3])
    F0, J0, G0, lam, sf, sg, Z, X, Fc, Gc = runs[True]
    assert np.abs(Z @ X - np.eye(n)).max() < 1e-9
    eF, eG = eq71(F0, J0, G0, Fc, Gc, X, sf, sg)
    assert eF < 1e-12 and eG < 1e-12, (eF, eG)
