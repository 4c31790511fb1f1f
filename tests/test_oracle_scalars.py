"""Pins for the oracle's scalar machinery: Philox, Lambert W0, rho0, tau (Eq. 7).

Each check compares against something other than the oracle's own formula:
published known-answer vectors, scipy's independent Lambert W, the paper's
printed constant, and the ODE of PAPER.md:1307-1320 (Corollary "Bounds on optimal rho" and its proof) that Eq. 7 solves.
"""
import math
import os

import numpy as np
import pytest
from scipy.special import lambertw

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _kat():
    rows = []
    with open(os.path.join(GOLDEN, "philox4x32_10_kat.txt")) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            v = [int(x, 16) for x in line.split()]
            rows.append((v[0:4], v[4:6], v[6:10]))
    return rows


def _consts():
    out = {}
    with open(os.path.join(GOLDEN, "paper_constants.txt")) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            name, val, tol = line.split()[:3]
            out[name] = ([float(x) for x in val.split(",")], float(tol))
    return out


@pytest.mark.parametrize("ctr,key,want", _kat())
def test_philox_known_answers(orc, ctr, key, want):
    assert list(orc.philox4x32_10(ctr, key)) == want


def test_pivot_uniform_construction(orc):
    # u = ((x0>>5) 2^26 + (x1>>6)) 2^-53 from the KAT block at ctr = key = 0 would be
    # 0.39904647231489565; the pivot stream uses ctr = (i, unit_lo, unit_hi, 'PIVT').
    x = orc.philox4x32_10([0, 0, 0, 0], [0, 0])
    u = ((int(x[0]) >> 5) * 2**26 + (int(x[1]) >> 6)) / 2**53
    assert u == pytest.approx(0.39904647231489565, abs=0)
    x = orc.philox4x32_10([7, 3, 0, 0x50495654], [42, 0])
    want = ((int(x[0]) >> 5) * 2**26 + (int(x[1]) >> 6)) / 2**53
    assert orc.pivot_uniform(42, 7, 3) == want
    us = np.array([orc.pivot_uniform(1, i, 0) for i in range(20000)])
    assert us.min() >= 0.0 and us.max() < 1.0
    assert abs(us.mean() - 0.5) < 0.01 and abs(us.var() - 1 / 12) < 0.005


def test_lambert_w0_residual_and_scipy(orc):
    zs = np.logspace(-8, 8, 1000)
    for z in zs:
        w = orc.lambert_w0(z)
        assert abs(w * math.exp(w) - z) <= 1e-12 * max(1.0, z), z
        ref = lambertw(z).real
        assert abs(w - ref) <= 1e-13 * max(1.0, abs(ref)), z
    ws = [orc.lambert_w0(z) for z in zs]
    assert all(b > a for a, b in zip(ws, ws[1:]))
    assert orc.lambert_w0(0.0) == 0.0
    c = _consts()
    assert abs(orc.lambert_w0(math.e) - c["lambertw_e"][0][0]) <= c["lambertw_e"][1]


def test_lambert_exponential_identity(orc):
    # exp(W0(z)) = z / W0(z)  (Lemma "Lambert W exponential")
    for z in np.logspace(-6, 6, 50):
        w = orc.lambert_w0(z)
        assert math.exp(w) == pytest.approx(z / w, rel=1e-12)


def test_rho0_paper_value(orc):
    c = _consts()
    want, tol = c["rho0"]
    assert abs(orc.rho0() - want[0]) <= tol
    # and to full precision against scipy's Lambert W
    ref = math.sqrt(1 + math.exp(lambertw(2 / math.e**2).real + 2))
    assert orc.rho0() == pytest.approx(ref, rel=1e-14)
    # Corollary proof: 2/(rho0^2+1) <= 1/5
    assert 2 / (orc.rho0() ** 2 + 1) <= 0.2


def test_temperature_fallback(orc):
    assert orc.temperature(0.1, 0.0, 3.0, 100) == 1.0
    assert orc.temperature(0.1, 2.0, 0.0, 100) == 1.0


def _rho(orc, beta, rq, rk, n):
    tau = orc.temperature(beta, rq, rk, n)
    return tau * tau * rq / rk  # rho = tau^2 R_Q / R_K


def test_temperature_solves_paper_ode(orc):
    # Eq. 7 gives rho = b/(2 W0(b/(2 rho0))) as a function of b = b0.  PAPER.md:1307-1320 (Corollary "Bounds on optimal rho" and its proof)
    # states this is the solution of d rho/db = rho/(2 rho + b), rho(0) = rho0.  Check the
    # ODE by central differences in b (varying n at fixed beta R_Q R_K), and the lower
    # bound rho >= rho0 (same Corollary).
    rq, rk, n = 3.0, 2.0, 4096
    rho0 = orc.rho0()

    def rho_at(b):  # choose beta so that b0 = log(n)/(beta R_Q R_K) + 2 equals b
        return _rho(orc, math.log(n) / ((b - 2.0) * rq * rk), rq, rk, n)

    for b in [2.5, 3.0, 5.0, 10.0, 40.0, 300.0]:
        h = 1e-4 * b
        r0 = rho_at(b)
        assert (rho_at(b + h) - rho_at(b - h)) / (2 * h) == pytest.approx(r0 / (2 * r0 + b), rel=1e-6)
        assert r0 >= rho0
    # b -> 0 limit of the closed form is rho0 (initial condition of the ODE)
    b = 1e-9
    assert b / (2 * orc.lambert_w0(b / (2 * rho0))) == pytest.approx(rho0, rel=1e-8)


def test_temperature_scale_covariance(orc):
    # rho depends on (R_Q, R_K) only through b0, i.e. through R_Q R_K.
    for c in [0.5, 2.0, 7.0]:
        assert _rho(orc, 0.1, 3.0 * c, 5.0 / c, 4096) == pytest.approx(_rho(orc, 0.1, 3.0, 5.0, 4096), rel=1e-13)


def test_temperature_n1(orc):
    # n = 1: b0 = 2, tau^2 = (R_K/R_Q) / W0(1/rho0)
    tau = orc.temperature(0.3, 2.0, 5.0, 1)
    want = (5.0 / 2.0) / lambertw(1 / orc.rho0()).real
    assert tau * tau == pytest.approx(want, rel=1e-13)
