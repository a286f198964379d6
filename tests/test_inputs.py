"""Checks of the seeded input generators (echo_inputs): determinism, recipe
numbers of DESIGN.md §5 / SURVEY App. A.  CPU only."""
import math

import numpy as np
import pytest

import echo_inputs as I


def test_splitmix_reference_values():
    # splitmix64 reference sequence for seed 0 (Vigna's published test vector prefix)
    r = I.SplitMix64(0)
    assert r.next() == 0xE220A8397B1DCDAF
    assert r.next() == 0x6E789E6AA1B965F4


def test_white_noise_range_and_determinism():
    a = I.white_noise(3, 10000)
    b = I.white_noise(3, 10000)
    assert np.array_equal(a, b)
    assert a.min() >= -1 and a.max() < 1 and abs(a.mean()) < 0.05
    assert not np.array_equal(a, I.white_noise(4, 10000))


def test_turbulence_recipe():
    p = I.problem(0)
    P8 = I.initial_prims(p)
    assert P8.shape == (8, 32, 32, 32)
    v = np.sqrt(P8[1] ** 2 + P8[2] ** 2 + P8[3] ** 2)
    assert v.max() <= 0.1
    assert np.abs(P8[0] - 1).max() <= 0.05 + 1e-15
    assert np.array_equal(P8, I.initial_prims(I.problem(0)))


def test_torus_recipe():
    # reading A15: r_in = 7M, r_max = 12M closes the torus; rho_max = 0.17575, r_out ~ 45.9
    p = I.problem(4)
    ell = I.torus_l_kepler(1.0, 0.9, 12.0)
    assert ell == pytest.approx(3.89900548995364, rel=1e-12)
    r = np.linspace(7.0, 60.0, 20001)
    rho, prs, v1, v3, inside = I.torus_hydro(p, r, np.full_like(r, math.pi / 2))
    assert rho.max() == pytest.approx(0.17575, rel=2e-4)
    assert r[np.argmax(rho)] == pytest.approx(12.0, abs=0.01)
    r_out = r[inside].max()
    assert r_out == pytest.approx(45.9, abs=0.1)


def test_cp_alfven_speed():
    assert I.cp_alfven_speed(0.1) == pytest.approx(0.407965001183163, rel=1e-13)
