"""GPU parity of ghsvd_reduce (Phase 2: JQR + QR of G P2) against the oracle's or_reduce.

Pivot choices depend on rounding of the J-dots (tree vs sequential sums), so the
factors are compared through what Phase 2 must preserve (eq 5.1 and PAPER.md:914-923):
the Grammians P2^T F~^* J~ F~ P2 = F^* J F and P2^T G~^* G~ P2 = G^* G with the GPU's
own P2, the structure (block upper triangular F, upper triangular G with real
non-negative diagonal), and the converged eigenvalues vs the oracle pipeline.
"""
import numpy as np
import pytest

import oracle
from paper_1907_08560_b200 import inputs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gh():
    from paper_1907_08560_b200 import build, ghsvd
    build.build()
    return ghsvd


MODES = {"planned": dict(unblocked=False), "colsearch": dict(unblocked=False, colsearch=True),
         "unblocked": dict(unblocked=True), "own_qr": dict(unblocked=False, own_qr=True)}


@pytest.mark.parametrize("mode", list(MODES))
@pytest.mark.parametrize("m,n,neg", [(60, 12, 0.5), (200, 40, 0.4), (150, 150, 0.5), (300, 64, 0.1), (97, 31, 0.5),
                                     (500, 300, 0.5), (400, 133, 0.3)])
def test_reduce_grammians(gh, m, n, neg, mode):
    """Every Phase-2 form (blocked with planned JQR pivots -- the default --, blocked with the
    pivots searched on the columns, unblocked: one reflector application per column; panels
    of <= 33 delayed reflectors, several panels and ragged last panels here)."""
    P = inputs.random_pencil(50 + m, m, n, neg)
    ctx = gh.Context(m, n)
    ctx.set_factors(P.F, P.J, P.G)
    ctx.reduce(**MODES[mode])
    # the blocked forms need the output-Z buffer (n x n) to hold the panel; thin problems run
    # the unblocked form whatever the flag (fallback_col -2)
    lds, ldn = -(-m // 16) * 16, -(-(n + 1) // 16) * 16   # phase2.cu's panel need vs the Z2 buffer
    blocked_fits = lds * 68 + 33 * 33 + 66 * n + 66 + ((m + 31) // 32 + 1) * 33 <= ldn * (n + 1)
    if mode == "planned":
        assert ctx.reduce_fallback_col == (-1 if blocked_fits else -2)
    F, J, G, p2 = ctx.get_factors()
    if n % 2:
        F, G, J = F[:-1, :-1], G[:-1, :-1], J[:-1]
    assert F.shape == (n, n) and sorted(p2) == list(range(n))
    H = P.F.conj().T @ (P.J[:, None] * P.F)
    S = P.G.conj().T @ P.G
    Hp, Sp = H[np.ix_(p2, p2)], S[np.ix_(p2, p2)]
    assert np.linalg.norm(F.conj().T @ (J[:, None] * F) - Hp) / np.linalg.norm(H) < 1e-11
    assert np.linalg.norm(G.conj().T @ G - Sp) / np.linalg.norm(S) < 1e-12
    assert np.abs(np.tril(G, -1)).max() == 0
    assert np.all(np.diag(G).real >= 0) and np.all(np.diag(G).imag == 0)
    npos = int((J > 0).sum())
    assert list(J) == [1] * npos + [-1] * (n - npos)
    # the oracle's JQR gives the same inertia and (usually) the same column pivoting
    Fs, Js, Gs, p2o, n2 = oracle.reduce(P.F, P.J, P.G)
    assert int((Js > 0).sum()) == npos
    ctx.close()


def test_config2_like_reduce_then_sweep(gh):
    """BASELINE configs[2] shape family (LAPW atoms, ~40 % negative), scaled down:
    factor -> reduce -> sweep vs the oracle pipeline (same factors after Phase 1)."""
    at = inputs.lapw_atoms(2, 4, 49, 256, 39 / 98)
    m, n = 2 * 4 * 49, 256
    ctx = gh.Context(m, n, 49)
    ctx.factor(at.A, at.B, at.U, at.TAA, at.TAB, at.TBB)
    ctx.reduce()
    F0, J0, G0, p2 = ctx.get_factors()
    st = ctx.sweep()
    lam, sf, sg, Z = ctx.extract()
    Fo, Jo, Go = oracle.factor(at.A, at.B, at.U, at.TAA, at.TAB, at.TBB)
    Fr, Gr, Zp, sto = oracle.hz_pointwise(Fo, Jo, Go)
    lo, *_ = oracle.extract(Fr, Jo, Gr, Zp)
    assert st["converged"]
    assert np.max(np.abs(np.sort(lam) - np.sort(lo)) / np.abs(np.sort(lo))) <= 1e-9
    # eigenvectors of the original (unreduced, unpermuted) pencil: residual
    Hx = Fo.conj().T @ (Jo[:, None] * (Fo @ Z))
    Sx = Go.conj().T @ (Go @ Z)
    nf2 = np.linalg.norm(Fo) ** 2 + np.linalg.norm(Go) ** 2
    res = np.linalg.norm(Hx - Sx * lam[None, :], axis=0) / (nf2 * np.linalg.norm(Z, axis=0))
    assert res.max() <= 1e-12 * n
    ctx.close()


@pytest.mark.parametrize("unblocked", [False, True])
@pytest.mark.parametrize("m,n,neg", [(200, 40, 0.4), (150, 150, 0.5), (97, 31, 0.5), (600, 257, 0.5)])
def test_reduce_colpiv_grammians(gh, m, n, neg, unblocked):
    """GHSVD_REDUCE_COLPIV: the QR of G P2 with column pivoting,
    F' = F P5.  The exported permutation is P2 P5: the Grammians are those of the original
    pencil under it, G' is upper triangular with a real non-negative, non-increasing
    diagonal (each pivot is the largest remaining column norm)."""
    P = inputs.random_pencil(70 + m, m, n, neg)
    ctx = gh.Context(m, n)
    ctx.set_factors(P.F, P.J, P.G)
    ctx.reduce(colpiv=True, unblocked=unblocked)
    F, J, G, p = ctx.get_factors()
    if n % 2:
        F, G, J = F[:-1, :-1], G[:-1, :-1], J[:-1]
    assert F.shape == (n, n) and sorted(p) == list(range(n))
    H = P.F.conj().T @ (P.J[:, None] * P.F)
    S = P.G.conj().T @ P.G
    Hp, Sp = H[np.ix_(p, p)], S[np.ix_(p, p)]
    assert np.linalg.norm(F.conj().T @ (J[:, None] * F) - Hp) / np.linalg.norm(H) < 1e-11
    assert np.linalg.norm(G.conj().T @ G - Sp) / np.linalg.norm(S) < 1e-12
    assert np.abs(np.tril(G, -1)).max() == 0
    d = np.diag(G)
    assert np.all(d.real >= 0) and np.all(d.imag == 0)
    assert np.all(np.diff(d.real) <= 1e-12 * d.real[0])
    ctx.close()


def test_colpiv_reduce_on_illconditioned_matches_tall(gh):
    """A config-3 analog (S singular values 1 ... 1e-12): the eigenvalues after the
    column-pivoted Phase 2 agree with the tall (Phase-2-skipped) computation to 1e-6
    (BASELINE's ill-conditioned tolerance), with residuals on the original pencil."""
    at = inputs.illcond_atoms(3, 4, 40, 128)
    m, n = 2 * 4 * 40, 128
    lams = {}
    for mode in ("tall", "colpiv"):
        ctx = gh.Context(m, n, 40, variant="bo")
        ctx.factor(at.A, at.B, at.U, at.TAA, at.TAB, at.TBB)
        if mode == "colpiv":
            ctx.reduce(colpiv=True)
        st = ctx.sweep()
        lam, sf, sg, Z = ctx.extract()
        ctx.close()
        assert st["converged"]
        lams[mode] = (lam, Z)
    a, b = np.sort(lams["tall"][0]), np.sort(lams["colpiv"][0])
    assert np.max(np.abs(a - b) / np.abs(a)) <= 1e-6
    Fo, Jo, Go = oracle.factor(at.A, at.B, at.U, at.TAA, at.TAB, at.TBB)
    lam, Z = lams["colpiv"]
    Hx = Fo.conj().T @ (Jo[:, None] * (Fo @ Z))
    Sx = Go.conj().T @ (Go @ Z)
    nf2 = np.linalg.norm(Fo) ** 2 + np.linalg.norm(Go) ** 2
    res = np.linalg.norm(Hx - Sx * lam[None, :], axis=0) / (nf2 * np.linalg.norm(Z, axis=0))
    assert res.max() <= 1e-12 * n


@pytest.mark.parametrize("colpiv", [False, True])
def test_blocked_and_unblocked_reduce_same_pencil(gh, colpiv):
    """LAPW atoms (config-2 family, ~40 % negative signs): the blocked and the unblocked
    Phase 2 may pivot differently on near-ties, but both reduce the same pencil -- the
    converged eigenvalues agree with each other and with the oracle's tall solve (1e-9)."""
    at = inputs.lapw_atoms(12, 4, 49, 300, 39 / 98)
    m, n = 2 * 4 * 49, 300
    lams = []
    for kw in MODES.values():
        ctx = gh.Context(m, n, 49, variant="bo")
        ctx.factor(at.A, at.B, at.U, at.TAA, at.TAB, at.TBB)
        ctx.reduce(colpiv=colpiv, **kw)
        st = ctx.sweep()
        lams.append(np.sort(ctx.extract(want_z=False)[0]))
        ctx.close()
        assert st["converged"]
    Fo, Jo, Go = oracle.factor(at.A, at.B, at.U, at.TAA, at.TAB, at.TBB)
    Fr, Gr, Zp, sto = oracle.hz_pointwise(Fo, Jo, Go)
    lo = np.sort(oracle.extract(Fr, Jo, Gr, Zp)[0])
    for lam in lams:
        assert np.max(np.abs(lam - lo) / np.abs(lo)) <= 1e-9


@pytest.mark.parametrize("m,n,neg,seed", [(300, 256, 0.4, 1), (500, 400, 0.5, 2), (200, 199, 0.5, 3)])
def test_planned_jqr_pivots_equal_column_search(gh, m, n, neg, seed):
    """The planned pivots are the paper's rule applied to the Schur complements of
    H = F^* J F, which equal the J-Grammians the column search reads: away from near-ties
    both choose the same interchanges and 1x1 / 2x2 pivots (same P2 and inertia)."""
    P = inputs.random_pencil(90 + seed, m, n, neg)
    out = {}
    for mode in ("planned", "colsearch"):
        ctx = gh.Context(m, n)
        ctx.set_factors(P.F, P.J, P.G)
        ctx.reduce(**MODES[mode])
        F, J, G, p2 = ctx.get_factors()
        out[mode] = (p2, int((J > 0).sum()), ctx.reduce_fallback_col)
        ctx.close()
    assert out["planned"][2] == -1 and out["colsearch"][2] == -2   # the plan ran, every pivot kept
    assert np.array_equal(out["planned"][0], out["colsearch"][0])
    assert out["planned"][1] == out["colsearch"][1]


def test_planned_jqr_on_illconditioned_config3_recipe(gh):
    """Config-3 recipe (S condition 1e12) at reduced size: the planned JQR keeps the
    Grammians and reduces the same pencil as the column search (converged lambda 1e-6)."""
    at = inputs.illcond_atoms(3, 8, 40, 256)
    m, n = 2 * 8 * 40, 256
    lams = []
    for mode in ("planned", "colsearch"):
        ctx = gh.Context(m, n, 40, variant="bo")
        ctx.factor(at.A, at.B, at.U, at.TAA, at.TAB, at.TBB)
        F0, J0, G0, _ = ctx.get_factors()
        ctx.reduce(**MODES[mode])
        F, J, G, p2 = ctx.get_factors()
        H0 = F0.conj().T @ (J0[:, None] * F0)
        assert np.linalg.norm(F.conj().T @ (J[:, None] * F) - H0[np.ix_(p2, p2)]) / np.linalg.norm(H0) < 1e-11
        st = ctx.sweep()
        lams.append(np.sort(ctx.extract(want_z=False)[0]))
        ctx.close()
        assert st["converged"]
    assert np.max(np.abs(lams[0] - lams[1]) / np.abs(lams[1])) <= 1e-6


def test_planned_pivots_fall_back_to_the_column_search(gh):
    """F and G of numerical rank n/2 plus a 1e-9 perturbation: after n/2 steps the Schur
    complements of the explicitly formed H = F^* J F and S = G^* G are ~1e-18 of the
    Grammians, below their rounding (~1e-16), so the planned pivots there are noise while
    the columns themselves still carry them to ~1e-7.  The check must reject them and the
    column search finish the factorization (R2-6): fallback_col >= 0, the Grammians
    preserved as by the column search throughout, the same inertia.  (Column grading alone
    does not do it: diagonally pivoted elimination is scaling-invariant.)"""
    m, n = 400, 256   # (square enough for the blocked form: the panel fits the n x n buffer)
    P = inputs.random_pencil(77, m, n, 0.5)
    rng = np.random.default_rng(5)

    def near_rank(X):
        r = n // 2
        A = X[:, :r] @ (rng.standard_normal((r, n)) + 1j * rng.standard_normal((r, n))) / np.sqrt(r)
        return np.asfortranarray(A + 1e-9 * X)

    F = near_rank(P.F)
    G = near_rank(P.G)
    H = F.conj().T @ (P.J[:, None] * F)
    S = G.conj().T @ G
    res = {}
    for mode in ("planned", "colsearch"):
        ctx = gh.Context(m, n)
        ctx.set_factors(F, P.J, G)
        ctx.reduce(colpiv=True, **MODES[mode])
        Fr, Jr, Gr, p = ctx.get_factors()
        res[mode] = (ctx.reduce_fallback_col, int((Jr > 0).sum()))
        eh = np.linalg.norm(Fr.conj().T @ (Jr[:, None] * Fr) - H[np.ix_(p, p)]) / np.linalg.norm(H)
        es = np.linalg.norm(Gr.conj().T @ Gr - S[np.ix_(p, p)]) / np.linalg.norm(S)
        assert eh < 1e-11 and es < 1e-12, (mode, eh, es)
        assert np.abs(np.tril(Gr, -1)).max() == 0
        ctx.close()
    assert res["planned"][0] >= 0          # the plan was stopped and the search took over
    assert res["planned"][1] == res["colsearch"][1]
