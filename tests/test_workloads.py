"""Input generators: the 12-point rule's exactness and the meshes' geometry (CPU)."""
import numpy as np
import pytest

from workloads import configs, geometry, rule


def _exact_monomial(a, b):
    # int over reference triangle (0,0),(1,0),(0,1) of x^a y^b = a! b! / (a+b+2)!
    from math import factorial
    return factorial(a) * factorial(b) / factorial(a + b + 2)


def test_rule12_degree6_exact():
    assert abs(rule.WEIGHTS.sum() - 1.0) < 1e-14
    x, y = rule.BARY[:, 1], rule.BARY[:, 2]
    for a in range(7):
        for b in range(7 - a):
            q = 0.5 * np.sum(rule.WEIGHTS * x ** a * y ** b)
            assert abs(q - _exact_monomial(a, b)) < 1e-14 * max(1.0, _exact_monomial(a, b) * 1e3)
    # and it is NOT exact at degree 7 (so the table is the degree-6 rule, not something else)
    errs = [abs(0.5 * np.sum(rule.WEIGHTS * x ** a * y ** (7 - a)) - _exact_monomial(a, 7 - a)) for a in range(8)]
    assert max(errs) > 1e-8


def test_disk_area_and_boundary():
    w = configs.config1(f="const")
    assert abs(w.M - 2000) <= 20
    assert w.N == 12 * w.M
    assert abs(w.weights.sum() - np.pi) < 1e-12          # smooth map: exact disk area
    assert np.all(w.weights > 0)
    assert np.all(np.hypot(w.nodes[..., 0], w.nodes[..., 1]) < 1.0)
    assert np.count_nonzero(w.curved) > 50


def test_square_meshes_area():
    w2 = configs.config2(n=30)
    assert abs(w2.weights.sum() - 1.0) < 1e-13
    # slivers exist with high aspect ratio
    t = w2.tri
    e = np.stack([np.hypot(*(t[:, (k + 1) % 3] - t[:, k]).T) for k in range(3)], 1)
    area = 0.5 * np.abs(np.cross(t[:, 1] - t[:, 0], t[:, 2] - t[:, 0]))
    aspect = e.max(1) ** 2 / (2 * area)
    assert aspect.max() > 100
    w4 = configs.config4(n=20, f_device="cpu")
    assert w4.M == 2 * 20 * 20
    assert abs(w4.weights.sum() - 1.0) < 1e-13


def test_full_size_counts():
    # sizes stated in BASELINE.json (config 2: 200k triangles incl. 5% cevian splits)
    w2 = configs.config2()
    assert abs(w2.M - 200_000) < 0.01 * 200_000


def test_curved_map_endpoints():
    # the blending map sends the curved edge onto the circle
    w = configs.config1(f="const")
    cur = np.nonzero(w.curved)[0][:20]
    lam = np.linspace(0, 1, 11)
    for m in cur:
        e = int(np.log2(w.curved[m] & -w.curved[m]))
        xi1 = np.zeros((1, lam.size)); xi2 = np.zeros((1, lam.size))
        # edge e = (v_e, v_{e+1}); barycentric l_e = 1 - lam, l_{e+1} = lam
        l = np.zeros((3, lam.size)); l[e] = 1 - lam; l[(e + 1) % 3] = lam
        xi1[0], xi2[0] = l[1], l[2]
        x, y = geometry.map_points(w.tri[m:m + 1], w.curved[m:m + 1], w.circle, xi1, xi2)
        assert np.allclose(np.hypot(x, y), 1.0, atol=1e-14)


def test_config3_generator_properties():
    """Scaled config 3: star-shaped, graded (area ratio > 1e3), nonconforming patches with gaps (total area
    slightly below the star's), positively oriented, no degenerate triangles, f vanishing at the boundary."""
    w = configs.config3(M_target=60000, lmin=7, lmax=13, g=0.1)
    t = w.tri
    area = 0.5 * ((t[:, 1, 0] - t[:, 0, 0]) * (t[:, 2, 1] - t[:, 0, 1]) - (t[:, 1, 1] - t[:, 0, 1]) * (t[:, 2, 0] - t[:, 0, 0]))
    assert np.all(area > 0)
    star_area = np.pi * (1.0 + 0.3 ** 2 / 2)       # (1/2) int (1 + 0.3 cos 5t)^2 dt
    assert star_area * 0.995 < area.sum() < star_area  # chords + gaps remove a little
    assert area.max() / area.min() > 1e3
    # every node lies inside the star
    r = np.hypot(w.nodes[..., 0], w.nodes[..., 1])
    th = np.arctan2(w.nodes[..., 1], w.nodes[..., 0])
    assert np.all(r < configs.star_radius(th))
    assert np.abs(w.f).max() > 0.99 and np.abs(w.f[r > 0.9]).max() < 1e-300
    # nonconforming: some vertices are not shared with any other triangle of a different patch (hanging
    # nodes / gaps), i.e. the vertex multiset has many singletons along patch seams
    v = np.round(t.reshape(-1, 2), 12)
    _, counts = np.unique(v, axis=0, return_counts=True)
    assert (counts == 1).sum() > 0
