"""Resumable sweeps: ghsvd_sweep keeps F', G', Z' (and W) between calls, so a solve split
into calls of C_max = c sweeps each (every call but the last returns NOT_CONVERGED) runs
exactly the same sequence of sweeps as one call -- bitwise the same eigenvalues, Z and X,
and the same total sweep count.  This is the resume path of a long solve (e.g. a serving
deadline per call)."""
import warnings

import numpy as np
import pytest

from paper_1907_08560_b200 import inputs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gh():
    from paper_1907_08560_b200 import build, ghsvd
    build.build()
    return ghsvd


@pytest.mark.parametrize("variant,chunk,want_x", [("pointwise", 1, False), ("pointwise", 4, True), ("bo", 1, False),
                                                  ("bo", 3, True), ("fb", 2, False)])
def test_chunked_sweeps_bitwise_equal_single_call(gh, variant, chunk, want_x):
    P = inputs.known_hyperbolic(41, 360, 224, 0.4)
    m, n = P.F.shape
    a = gh.Context(m, n, variant=variant, max_sweeps=64, want_x=want_x)
    a.set_factors(P.F, P.J, P.G)
    sa = a.sweep()
    la, _, _, Za = a.extract()
    Xa = a.extract_x() if want_x else None
    b = gh.Context(m, n, variant=variant, max_sweeps=chunk, want_x=want_x)
    b.set_factors(P.F, P.J, P.G)
    total, calls = 0, 0
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")   # NOT_CONVERGED after every call but the last
        while True:
            st = b.sweep()
            total += st["sweeps"]
            calls += 1
            if st["converged"] or calls > 64:
                break
    lb, _, _, Zb = b.extract()
    Xb = b.extract_x() if want_x else None
    assert sa["converged"] and st["converged"]
    assert total == sa["sweeps"] and calls == -(-sa["sweeps"] // chunk)
    np.testing.assert_array_equal(la, lb)
    np.testing.assert_array_equal(Za, Zb)
    if want_x:
        np.testing.assert_array_equal(Xa, Xb)
    a.close()
    b.close()


@pytest.mark.parametrize("variant,want_x,n", [("pointwise", False, 224), ("bo", True, 224), ("bo", False, 191),
                                              ("fb", False, 160)])
def test_checkpoint_restore_in_new_context(gh, variant, want_x, n):
    """ghsvd_get_state after k sweeps, destroy, a NEW context with the same problem set up
    (set_factors), ghsvd_set_state, sweep to convergence: bitwise the uninterrupted solve
    (odd n: the bordered state round-trips too)."""
    P = inputs.known_hyperbolic(42, n + 130, n, 0.4)
    m = P.F.shape[0]
    a = gh.Context(m, n, variant=variant, max_sweeps=64, want_x=want_x)
    a.set_factors(P.F, P.J, P.G)
    sa = a.sweep()
    la, _, _, Za = a.extract()
    Xa = a.extract_x() if want_x else None
    a.close()
    b = gh.Context(m, n, variant=variant, max_sweeps=3, want_x=want_x)
    b.set_factors(P.F, P.J, P.G)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        s1 = b.sweep()
    assert not s1["converged"]
    ck = b.get_state()
    b.close()
    c = gh.Context(m, n, variant=variant, max_sweeps=64, want_x=want_x)
    c.set_factors(P.F, P.J, P.G)
    c.set_state(ck)
    s2 = c.sweep()
    lc, _, _, Zc = c.extract()
    Xc = c.extract_x() if want_x else None
    c.close()
    assert s2["converged"] and s1["sweeps"] + s2["sweeps"] == sa["sweeps"]
    np.testing.assert_array_equal(la, lc)
    np.testing.assert_array_equal(Za, Zc)
    if want_x:
        np.testing.assert_array_equal(Xa, Xc)


def test_set_state_requires_a_problem(gh):
    c = gh.Context(64, 32)
    with pytest.raises(gh.GHSVDError) as e:
        c.set_state({"F": np.zeros((64, 32), complex), "G": np.zeros((64, 32), complex),
                     "Z": np.eye(32, dtype=complex), "W": None})
    assert e.value.status == -2
    c.close()
