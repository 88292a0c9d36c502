"""Host-side layout of factors given to ghsvd_set_factors, so the oracle gets its inputs
from the test's own data, never from the CUDA path (ghsvd_get_factors).

The device keeps F's rows stably sorted by J (+ first) and G's rows as given
(include/ghsvd.h, ghsvd_set_factors); an odd n is bordered by one row and one
column holding a single 1 in F and G, the border row last with J = -1 (reading C-10).
This is data layout only (a permutation and an appended unit row/column), restated here
from the documented contract; test_set_get_factors_sorts_rows_by_J checks that the device
agrees with it bitwise."""
import numpy as np


def device_layout(F, J, G):
    """(F, J, G) as the sweep sees them after set_factors: F rows J-sorted (stable), G as
    given, odd n bordered.  Returns Fortran-ordered copies."""
    F = np.asarray(F, dtype=np.complex128)
    G = np.asarray(G, dtype=np.complex128)
    J = np.asarray(J, dtype=np.int8)
    perm = np.argsort(-J.astype(np.int64), kind="stable")
    F, J = F[perm], J[perm]
    m, n = F.shape
    if n % 2:
        Fb = np.zeros((m + 1, n + 1), np.complex128)
        Gb = np.zeros((m + 1, n + 1), np.complex128)
        Fb[:m, :n], Gb[:m, :n] = F, G
        Fb[m, n] = Gb[m, n] = 1.0
        F, G, J = Fb, Gb, np.concatenate([J, np.array([-1], np.int8)])
    return np.asfortranarray(F), J.copy(), np.asfortranarray(G)
