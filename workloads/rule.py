"""12-point degree-6 symmetric triangle quadrature rule (input data, not method arithmetic).

The paper discretises the domain as a union of triangles, each carrying a
p-point rule (§2.2: "each triangle T_j is equipped with
a p-point quadrature rule of order q_v ... N = Mp").  BASELINE.json fixes the
rule for every config: the 12-point symmetric rule of Dunavant (1985), exact
for polynomials of degree <= 6.  The structure is two
S21 orbits and one S111 orbit in barycentric coordinates; weights sum to 1 and
are multiplied by the (mapped) triangle area.

Degree-6 exactness is pinned in tests/test_workloads.py against exact monomial
integrals on the reference triangle.
"""
import numpy as np

_S21 = [  # (a, weight): points (a, a, 1-2a) and permutations
    (0.249286745170910, 0.116786275726379),
    (0.063089014491502, 0.050844906370207),
]
_S111 = [  # (a, b, c, weight): all 6 permutations
    (0.053145049844817, 0.310352451033784, 0.636502499121399, 0.082851075618374),
]


def _build():
    bary, wts = [], []
    for a, w in _S21:
        b = 1.0 - 2.0 * a
        for p in [(a, a, b), (a, b, a), (b, a, a)]:
            bary.append(p)
            wts.append(w)
    for a, b, c, w in _S111:
        for p in [(a, b, c), (a, c, b), (b, a, c), (b, c, a), (c, a, b), (c, b, a)]:
            bary.append(p)
            wts.append(w)
    bary = np.array(bary, dtype=np.float64)
    # re-normalise each barycentric triple so it sums to exactly 1 in fp64
    bary[:, 0] = 1.0 - bary[:, 1] - bary[:, 2]
    return bary, np.array(wts, dtype=np.float64)


BARY, WEIGHTS = _build()          # (12, 3), (12,) ; sum(WEIGHTS) == 1 (to 1e-15)
P = 12
