"""GPU: proj/tests/test_geo.cpp ported onto the device haversine (kernel (1)
arithmetic), plus agreement with the reference's glibc haversine."""
import math

import numpy as np
import pytest

import oracle_harness as H
from paper_2001_05291_b200 import fleetplace as F

pytestmark = pytest.mark.gpu
R = F.kEarthRadiusKm


def great_circle_km(a, b, r):
    """proj/tests/test_oracles.hpp:19-37: the atan2/unit-vector route."""
    d = math.pi / 180.0
    la1, lo1, la2, lo2 = a[0] * d, a[1] * d, b[0] * d, b[1] * d
    x1, y1, z1 = math.cos(la1) * math.cos(lo1), math.cos(la1) * math.sin(lo1), math.sin(la1)
    x2, y2, z2 = math.cos(la2) * math.cos(lo2), math.cos(la2) * math.sin(lo2), math.sin(la2)
    cx, cy, cz = y1 * z2 - z1 * y2, z1 * x2 - x1 * z2, x1 * y2 - y1 * x2
    return r * math.atan2(math.sqrt(cx * cx + cy * cy + cz * cz), x1 * x2 + y1 * y2 + z1 * z2)


def test_identical_points():
    assert F.haversine_km((43.7, -79.4), (43.7, -79.4)) == 0.0


def test_analytic_references():
    anti = F.haversine_km((0.0, 0.0), (0.0, 180.0))
    assert abs(anti - math.pi * R) <= 1e-6 * anti
    assert abs(anti - 20015.114442035924) <= 1e-6 * anti
    q = F.haversine_km((0.0, 0.0), (90.0, 0.0))
    assert abs(q - math.pi * R / 2) <= 1e-6 * q
    assert abs(q - 10007.557221017962) <= 1e-6 * q


def test_cross_checked_fixed_pair():
    assert abs(F.haversine_km((45.0, -75.0), (50.0, -85.0)) - 933.2885511911311) <= 1e-12 * 933.29


def test_vector_route_oracle_and_symmetry_and_triangle():
    rng = np.random.default_rng(20240601)
    n = 2000
    a = (rng.uniform(-90, 90, n), rng.uniform(-180, 180, n))
    b = (rng.uniform(-90, 90, n), rng.uniform(-180, 180, n))
    c = (rng.uniform(-90, 90, n), rng.uniform(-180, 180, n))
    ab = F.haversine_km_batch(*a, *b)
    ba = F.haversine_km_batch(*b, *a)
    aa = F.haversine_km_batch(*a, *a)
    ac = F.haversine_km_batch(*a, *c)
    bc = F.haversine_km_batch(*b, *c)
    assert np.array_equal(ab, ba)                      # exact symmetry
    assert (aa == 0.0).all()
    assert (ab >= 0).all() and (ab <= math.pi * R).all()
    assert (ac <= ab + bc + 1e-6).all()                # triangle inequality
    for k in range(250):
        ref = great_circle_km((a[0][k], a[1][k]), (b[0][k], b[1][k]), R)
        assert abs(ab[k] - ref) <= 1e-9 * max(ref, 1.0)
    for k in range(n):
        # the reference's own (glibc) haversine: bit-identical
        r2 = H.REF.ref_haversine_km(a[0][k], a[1][k], b[0][k], b[1][k], R)
        assert ab[k] == r2, (k, ab[k], r2)


def test_mission_cost_sums_the_two_legs():
    base, pickup, delivery = (44.0, -79.0), (45.0, -78.0), (43.0, -80.0)
    assert F.mission_cost_km(base, pickup, delivery) == \
        F.haversine_km(base, pickup) + F.haversine_km(base, delivery)
    assert F.mission_cost_km(base, base, base) == 0.0
    assert abs(F.mission_cost_km(base, pickup, pickup) - 2 * F.haversine_km(base, pickup)) <= 1e-12 * 300
    dlat = 0.0899320363724538
    assert abs(F.mission_cost_km((0.0, 0.0), (dlat, 0.0), (-dlat, 0.0)) - 20.0) <= 1e-9 * 20


def test_validity_bounds():
    assert F.valid((45.0, -75.0)) and F.valid((-90.0, 180.0))
    assert not F.valid((91.0, 0.0)) and not F.valid((0.0, -180.5))
