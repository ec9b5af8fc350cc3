"""Function-level parity and properties of the device arithmetic, through the
C-ABI checks ef_eval_dij / ef_eval_limiter (the stage kernels' own device code).

* bitwise equal to the unmodified reference's riemann.d_ij_low and
  limiter.limiter_compute on the seeded batches of tests/golden/functions_*.npz
  (extreme density/pressure ratios, identical states, equal pressures, zero and
  antisymmetric c vectors; Newton steps 2 and 4), and to the oracle on fresh
  random batches;
* the reference's unit-test properties (test_riemann.py:23-30, :87-98;
  test_limiter.py:86-102, :153-158): the identical-state pair gives
  (|u.n| + c)|c|, d is symmetric, l lies in [0, 1] and U + l P keeps the
  density inside the bounds."""

import os

import numpy as np
import pytest

import oracle as O
from goldens import GOLDEN_DIR
from paper_2007_00094_b200.physics import AIR
from paper_2007_00094_b200.stepper import eval_arith, eval_dij, eval_limiter

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dim", [2, 3])
def test_device_functions_match_reference(dim):
    z = np.load(os.path.join(GOLDEN_DIR, f"functions_{dim}d.npz"))
    d, bad = eval_dij(z["Ui"], z["Uj"], z["cij"], z["cji"])
    assert not bad.any()
    assert np.array_equal(d, z["d"])
    for newton in (2, 4):
        l = eval_limiter(z["U"], z["P"], z["bounds"], newton)
        assert np.array_equal(l, z[f"l_newton{newton}"])


def _states(rng, n, dim):
    rho = np.exp(rng.uniform(np.log(1e-6), np.log(1e3), n))
    u = rng.normal(0.0, 5.0, (n, dim))
    p = np.exp(rng.uniform(np.log(1e-8), np.log(1e8), n))
    U = np.empty((n, dim + 2))
    U[:, 0] = rho
    U[:, 1:-1] = rho[:, None] * u
    U[:, -1] = p / AIR.gm1 + 0.5 * rho * (u * u).sum(axis=1)
    return U


@pytest.mark.parametrize("scale", [0.3, 3e-2, 1e-3, 1e-6, 1e-12])
def test_device_dij_near_states_equals_oracle(scale):
    """Neighbouring states of a smooth flow: U_j = U_i perturbed by `scale`
    (relative) in density, velocity and pressure, with c_ji = -c_ij perturbed.
    Here the 3D path decides most pairs without the exact two-rarefaction p*
    (lambda_fast: certified enclosure of p*, wave-dominance test), and many pairs
    sit at the decision boundaries (p* ~ p_i ~ p_j, psi(p_max) ~ 0).  Bitwise
    equal to the oracle (the reference's operation sequence)."""
    dim = 3
    rng = np.random.default_rng(int(1e6 * scale) + 5)
    n = 400000
    rho = np.exp(rng.uniform(np.log(0.1), np.log(10.0), n))
    u = rng.normal(0.0, 1.0, (n, dim))
    p = np.exp(rng.uniform(np.log(0.1), np.log(10.0), n))

    def cons(rho, u, p):
        U = np.empty((len(rho), dim + 2))
        U[:, 0] = rho
        U[:, 1:-1] = rho[:, None] * u
        U[:, -1] = p / AIR.gm1 + 0.5 * rho * (u * u).sum(axis=1)
        return U

    Ui = cons(rho, u, p)
    Uj = cons(rho * np.exp(scale * rng.normal(size=n)), u + scale * rng.normal(size=(n, dim)),
              p * np.exp(scale * rng.normal(size=n)))
    cij = rng.normal(0.0, 1.0, (n, dim))
    cji = -cij * (1 + 1e-3 * rng.normal(size=(n, 1)))
    d, bad = eval_dij(Ui, Uj, cij, cji)
    do, bo = O.eval_dij(Ui, Uj, cij, cji)
    assert not bo.any()
    assert np.array_equal(bad, bo)
    assert np.array_equal(d.view(np.int64), do.view(np.int64))


@pytest.mark.parametrize("dim", [2, 3])
def test_device_dij_equals_oracle_on_random_batches(dim):
    rng = np.random.default_rng(11 + dim)
    n = 200000
    Ui, Uj = _states(rng, n, dim), _states(rng, n, dim)
    cij, cji = rng.normal(0.0, 1.0, (n, dim)), rng.normal(0.0, 1.0, (n, dim))
    d, bad = eval_dij(Ui, Uj, cij, cji)
    do, bo = O.eval_dij(Ui, Uj, cij, cji)
    assert np.array_equal(d, do) and np.array_equal(bad, bo)
    # symmetry (test_riemann.py:87-98)
    d2, _ = eval_dij(Uj, Ui, cji, cij)
    assert np.array_equal(d, d2)


@pytest.mark.parametrize("dim", [2, 3])
def test_identical_states_give_wave_speed(dim):
    """test_riemann.py:23-30: for U_i = U_j the bound is |u.n| + c, times |c|."""
    rng = np.random.default_rng(5)
    n = 10000
    # moderate Mach numbers: p recovered from E without cancellation
    rho = np.exp(rng.uniform(np.log(1e-2), np.log(1e2), n))
    u = rng.normal(0.0, 1.0, (n, dim))
    p = np.exp(rng.uniform(np.log(1e-1), np.log(1e1), n)) * rho
    U = np.empty((n, dim + 2))
    U[:, 0] = rho
    U[:, 1:-1] = rho[:, None] * u
    U[:, -1] = p / AIR.gm1 + 0.5 * rho * (u * u).sum(axis=1)
    c = rng.normal(0.0, 1.0, (n, dim))
    d, _ = eval_dij(U, U, c, -c)
    cs = np.sqrt(AIR.gamma * p / rho)
    nrm = np.linalg.norm(c, axis=1)
    expect = (np.abs((u * c).sum(axis=1) / nrm) + cs) * nrm
    assert np.allclose(d, expect, rtol=1e-11, atol=0.0)


@pytest.mark.parametrize("dim", [2, 3])
def test_limiter_properties_and_parity(dim):
    """l in [0, 1], density of U + l P inside [rho_min, rho_max] (test_limiter.py:
    153-158), Psi(U + l P) >= -tol (:86-102); equal to the oracle bitwise."""
    rng = np.random.default_rng(23 + dim)
    n = 100000
    U = _states(rng, n, dim)
    P = rng.normal(0.0, 1.0, (n, dim + 2)) * U * np.exp(rng.uniform(-4, 2, n))[:, None]
    rho = U[:, 0]
    rmin = rho * (1.0 - rng.uniform(0.0, 0.5, n))
    rmax = rho * (1.0 + rng.uniform(0.0, 0.5, n))
    eps = U[:, -1] - 0.5 * (U[:, 1:-1] ** 2).sum(axis=1) / rho
    pmin = eps * rho ** (-AIR.gamma) * (1.0 - rng.uniform(0.0, 0.2, n))
    bounds = np.column_stack([rmin, rmax, pmin])
    for newton in (1, 2, 4):
        l = eval_limiter(U, P, bounds, newton)
        assert np.array_equal(l, O.eval_limiter(U, P, bounds, newton))
        assert np.all((l >= 0.0) & (l <= 1.0))
        r = rho + l * P[:, 0]
        assert np.all(r >= rmin * (1 - 1e-12)) and np.all(r <= rmax * (1 + 1e-12))


def test_limiter_fast_accept_bound_is_an_upper_bound():
    """The limiter's fast accept (ef_math.cuh: pow_ub) must bound the exact pow
    from above on its whole range, and tightly (within 2^-12)."""
    from paper_2007_00094_b200 import _lib
    from paper_2007_00094_b200.stepper import shared_pow

    rng = np.random.default_rng(11)
    x = np.concatenate([2.0 ** rng.uniform(-20, 20, 2_000_000), 1.0 + rng.uniform(-1e-6, 1e-6, 200_000),
                        np.nextafter(2.0 ** -20, 1.0) * (1 + rng.uniform(0, 1e-3, 1000)),
                        np.nextafter(2.0 ** 20, 0.0) * (1 - rng.uniform(0, 1e-3, 1000))])
    for y in (AIR.gamma + 1.0, AIR.gamma, 1.0, 4.0):
        ub = np.empty_like(x)
        assert _lib.load().ef_pow_bound_device(x.ctypes.data, float(y), ub.ctypes.data, x.size) == 0
        exact = shared_pow(x, y)
        assert np.all(ub >= exact), (y, np.min(ub / exact))
        assert np.max(ub / exact) < 1.0 + 2.0 ** -12
    out = np.empty(4)
    xs = np.array([2.0 ** -21, 2.0 ** 21, 0.0, np.nan])
    _lib.load().ef_pow_bound_device(xs.ctypes.data, 2.4, out.ctypes.data, 4)
    assert np.all(np.isinf(out))


def _bit_patterns(rng, n):
    """Doubles with exponents in the safe range and adversarial significands: random bits,
    all ones / all zeros tails, neighbours of powers of two and of squares."""
    sig = rng.integers(0, 1 << 52, n, dtype=np.uint64)
    kind = rng.integers(0, 8, n)
    tail = rng.integers(1, 52, n).astype(np.uint64)
    ones = (np.uint64(1) << tail) - np.uint64(1)
    sig = np.where(kind == 0, sig | ones, sig)                       # trailing ones
    sig = np.where(kind == 1, sig & ~ones, sig)                      # trailing zeros
    sig = np.where(kind == 2, ones, sig)                             # just above a power of two
    sig = np.where(kind == 3, np.uint64((1 << 52) - 1) ^ ones, sig)  # just below the next one
    e = rng.integers(1023 - 450, 1023 + 450, n).astype(np.uint64)
    sign = rng.integers(0, 2, n).astype(np.uint64)
    return ((sign << np.uint64(63)) | (e << np.uint64(52)) | sig).view(np.float64)


def test_straight_line_division_and_root_are_ieee():
    """rcp_sl / div_sl / sqrt_sl / qdiv_sl (ef_math.cuh) restate nvcc's fast paths of 1/b, a/b,
    sqrt: no operand in the safe range may differ in a bit (the reference divides and takes
    roots with numpy's IEEE operations, riemann.py:56-109)."""
    rng = np.random.default_rng(20070094)
    total = np.zeros(4, dtype=np.uint64)
    for _ in range(4):
        n = 1 << 24
        a, b = _bit_patterns(rng, n), _bit_patterns(rng, n)
        # quotients near 1 and exact squares / products stress the final rounding
        k = n // 4
        b[:k] = a[:k] * (1.0 + rng.integers(-4, 5, k) * 2.0 ** -52)
        r = np.abs(_bit_patterns(rng, k))
        a[k:2 * k] = np.where(np.isfinite(r * r) & (r * r > 0), r * r, a[k:2 * k])
        total += eval_arith(a, b)
    assert not total.any(), total


@pytest.mark.parametrize("dim", [2, 3])
def test_device_dij_corner_cases_equal_oracle(dim):
    """Pairs that leave the straight-line path (or sit on its selects): zero momenta and
    momenta along / across the normal, equal pressures, strong shocks and expansions up to
    vacuum, extreme magnitudes, inadmissible states."""
    rng = np.random.default_rng(77 + dim)
    n = 60000
    Ui, Uj = _states(rng, n, dim), _states(rng, n, dim)
    cij = rng.normal(0.0, 1.0, (n, dim))
    cji = -cij * (1 + 1e-3 * rng.normal(size=(n, 1)))
    k = n // 12
    s = [slice(q * k, (q + 1) * k) for q in range(12)]
    Ui[s[0], 1:-1] = 0.0                                        # i at rest
    Ui[s[1], 1:-1] = 0.0
    Uj[s[1], 1:-1] = 0.0                                        # both at rest
    cij[s[2], 1:] = 0.0                                         # axis-aligned normals
    cji[s[2], 1:] = 0.0
    Ui[s[2], 2:-1] = 0.0                                        # momentum along the normal: tt = 0
    Uj[s[3]] = Ui[s[3]]                                         # equal pressures, opposite velocities
    Uj[s[3], 1:-1] = -Ui[s[3], 1:-1]
    Uj[s[4], 1:-1] += 30.0 * Uj[s[4], :1] * cij[s[4]] / np.linalg.norm(cij[s[4]], axis=1, keepdims=True)  # vacuum
    Uj[s[5], 1:-1] -= 30.0 * Uj[s[5], :1] * cij[s[5]] / np.linalg.norm(cij[s[5]], axis=1, keepdims=True)  # two shocks
    Uj[s[6], -1] *= 1e6                                         # pressure ratio 1e6
    Ui[s[7]] *= 1e60                                            # large magnitudes
    Uj[s[7]] *= 1e60
    Ui[s[8]] *= 1e-70                                           # small magnitudes
    Uj[s[8]] *= 1e-70
    Uj[s[9], -1] = 0.5 * (Uj[s[9], 1:-1] ** 2).sum(axis=1) / Uj[s[9], 0] * (1 - 1e-3)  # p < 0
    Uj[s[10], 0] = -Uj[s[10], 0]                                # rho < 0
    cji[s[11]] = 0.0                                            # a zero-norm direction
    with np.errstate(all="ignore"):
        d, bad = eval_dij(Ui, Uj, cij, cji)
        do, bo = O.eval_dij(Ui, Uj, cij, cji)
    assert np.array_equal(bad, bo) and bo[s[9]].all() and bo[s[10]].all() and not bo[s[0]].any()
    good = bo == 0  # a flagged pair raises; its value is not used
    assert np.array_equal(d[good].view(np.int64), do[good].view(np.int64))


@pytest.mark.parametrize("dim", [2, 3])
def test_device_dij_psi_sign_near_ties_equal_oracle(dim):
    """The straight-line path decides the sign of psi = f_lo + du (riemann.py:103) from an
    approximation with a certified margin (ef_math.cuh: lambda_sl) and leaves near-ties to
    the general code: pairs whose velocity jump cancels the shock function to a relative
    1e-6 ... one ulp, and equal-pressure pairs (f_lo = +0: the sign is du's) with
    compressive, expansive and zero velocity jumps."""
    rng = np.random.default_rng(401 + dim)
    n = 40000
    g = AIR.gamma
    rhoL, rhoR = np.exp(rng.uniform(-2, 2, n)), np.exp(rng.uniform(-2, 2, n))
    pL, pR = np.exp(rng.uniform(-2, 2, n)), np.exp(rng.uniform(-2, 2, n))
    eq = np.arange(n) % 4 == 0
    pR[eq] = pL[eq]
    lo = pL < pR
    p_lo, p_hi, rho_lo = np.where(lo, pL, pR), np.where(lo, pR, pL), np.where(lo, rhoL, rhoR)
    F = np.sqrt(2.0) * (p_hi - p_lo) / np.sqrt(rho_lo * ((g + 1.0) * p_hi + (g - 1.0) * p_lo))
    eps = rng.choice([0.0, 1e-16, -1e-16, 3e-16, -3e-16, 1e-13, -1e-13, 1e-10, -1e-10, 1e-6, -1e-6], n)
    du = -F * (1.0 + eps)
    du[eq] = rng.choice([0.0, -0.3, 0.3, -1e-12, 1e-12], int(eq.sum()))
    uL = rng.normal(0.0, 0.5, n)
    uR = uL + du
    nrm = rng.normal(0.0, 1.0, (n, dim))
    nrm[: n // 2, 1:] = 0.0  # axis-aligned: the projections carry u exactly
    nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
    t = rng.normal(0.0, 0.3, (n, dim))
    t -= (t * nrm).sum(axis=1, keepdims=True) * nrm  # a common tangential velocity
    t[: n // 2] = 0.0

    def state(rho, u, p):
        v = u[:, None] * nrm + t
        U = np.empty((n, dim + 2))
        U[:, 0] = rho
        U[:, 1:-1] = rho[:, None] * v
        U[:, -1] = p / AIR.gm1 + 0.5 * rho * (v * v).sum(axis=1)
        return U

    Ui, Uj = state(rhoL, uL, pL), state(rhoR, uR, pR)
    cij = nrm * np.exp(rng.uniform(-8, 0, n))[:, None]
    d, bad = eval_dij(Ui, Uj, cij, -cij)
    do, bo = O.eval_dij(Ui, Uj, cij, -cij)
    assert not bo.any() and np.array_equal(bad, bo)
    assert np.array_equal(d.view(np.int64), do.view(np.int64))
