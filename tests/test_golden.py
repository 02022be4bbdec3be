"""Paper-stated values (tests/golden/paper_values.json, each entry citing PAPER.md) against the CPU oracle and the
library's host-side method math (CPU only)."""
import json
import math
import os

import numpy as np

import oracle

HERE = os.path.dirname(os.path.abspath(__file__))
G = {e["name"]: e for e in json.load(open(os.path.join(HERE, "golden", "paper_values.json")))["entries"]}


def _mono(a, b):
    d = a + b
    return d * (d + 1) // 2 + (d - a)


def test_W_limit():
    e = G["W_limit_R_2sqrt2"]
    assert abs(float(oracle.WR(0.0, e["R"])) - e["value"]) < e["tol"]
    assert abs((1 - 2 * math.log(2 * math.sqrt(2))) * 8 / 4 - e["value"]) < e["tol"]


def test_local_kernel_decay():
    e = G["local_kernel_decay_at_12_sqrt_delta"]
    z = e["r_over_sqrt_delta"] ** 2 / 4.0
    assert float(oracle.e1(z)) / (4 * math.pi) < e["upper_bound"]


def test_on_boundary_coefficients_library():
    import paper_2409_11998_b200 as vp
    e = G["on_boundary_VL_coefficients"]
    b, c = vp.debug_local_coef("circle", [0, 0, 1.0 / e["kappa"], 0], 1.0 / e["kappa"], 0.0, e["delta"], 2, 6)
    assert b
    assert abs(c[_mono(0, 0)] - e["coef_f"]) < 1e-15
    # the inward normal at (1/kappa, 0) is -x: f_eta = -f_x, so the a10 coefficient is -coef_f_eta
    assert abs(c[_mono(1, 0)] + e["coef_f_eta"]) < 1e-16
    # Lap f = 2 a20 + 2 a02
    assert abs(c[_mono(2, 0)] - 2 * e["coef_lap"]) < 1e-18 and abs(c[_mono(0, 2)] - 2 * e["coef_lap"]) < 1e-18


def test_interior_constant_f_library():
    import paper_2409_11998_b200 as vp
    e = G["interior_VL_constant_f"]
    b, c = vp.debug_local_coef("none", [0, 0, 0, 0], 0.5, 0.5, e["delta"], 3, 6)
    assert not b and c[0] == e["value"]


def test_near_history_multiplier_k0_library():
    import paper_2409_11998_b200 as vp
    e = G["heat_split_at_delta2_over_delta1_32"]
    assert abs(vp.debug_mult(0, 0.0, e["delta1"], 32 * e["delta1"]) - e["value_k0"]) < 1e-16
