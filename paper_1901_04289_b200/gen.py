"""Deterministic synthetic inputs for the BASELINE.json configs.

There is no public benchmark suite for this path: the reference measures on
seeded random balls (src/bench.cpp:24-171).  These generators produce the
configs' shapes and value distributions from a fixed numpy PCG64 seed; the
same arrays feed the GPU path, the reference (oracle/_ref) and the C
restatement, so all three see identical bits.

Conventions:
* a "p-bit mantissa in [0.5,1)" is ceil(p/64) random limbs with the top bit
  forced on and the bits below p cleared; zero low limbs shrink the limb count
  exactly as apfloat_normalize does (src/apfloat.cpp:116-136) because the SoA
  layout stores mantissas top-aligned;
* "exponent e" is the ApFloat exponent (value in [2^(e-1), 2^e));
* "radius 2^-k |m|" is mag_upper_from_apfloat(m).mul_2exp(-k)
  (src/mag.cpp:147-153, 89-97).
"""
from __future__ import annotations

import numpy as np

from .balls import APB_FINITE, APB_SIGN, APB_ZERO, BallArray, limbs_for

SEED_BASE = 0xB200C0F1


def rng_for(config: int, salt: int = 0) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(SEED_BASE + 1000 * config + salt))


def random_mantissas(rng: np.random.Generator, count: int, p: int) -> np.ndarray:
    L = limbs_for(p)
    m = rng.integers(0, np.iinfo(np.uint64).max, size=(count, L), dtype=np.uint64, endpoint=True)
    m[:, L - 1] |= np.uint64(1 << 63)
    cut = 64 * L - p
    if cut:
        m[:, 0] &= ~np.uint64((1 << cut) - 1)
    return m


def rad_from_mid(mant: np.ndarray, exp: np.ndarray, k: int):
    """Mag of 2^-k * upper(|m|): b = top30(m) + 1 (canonicalized), f = e - k"""
    top = mant[:, -1]
    b = (top >> np.uint64(34)) + np.uint64(1)
    f = exp.astype(np.int64) - np.int64(k)
    carry = b == np.uint64(1 << 30)
    b = np.where(carry, np.uint64(1 << 29), b)
    f = np.where(carry, f + 1, f)
    return b.astype(np.uint32), f.astype(np.int64)


def random_balls(rng: np.random.Generator, count: int, p: int, exps: np.ndarray | None = None,
                 e_lo: int = 0, e_hi: int = 0, rad_k: int | None = None,
                 zero_frac: float = 0.0, rad_frac: float = 1.0) -> BallArray:
    mant = random_mantissas(rng, count, p)
    if exps is None:
        exps = rng.integers(e_lo, e_hi, size=count, endpoint=True, dtype=np.int64)
    exps = np.asarray(exps, np.int64)
    neg = rng.integers(0, 2, size=count, dtype=np.uint8).astype(bool)
    kind = np.where(neg, APB_FINITE | APB_SIGN, APB_FINITE).astype(np.uint8)
    rad_man = np.zeros(count, np.uint32)
    rad_exp = np.zeros(count, np.int64)
    if rad_k is not None:
        b, f = rad_from_mid(mant, exps, rad_k)
        has = np.ones(count, bool) if rad_frac >= 1.0 else rng.random(count) < rad_frac
        rad_man = np.where(has, b, 0).astype(np.uint32)
        rad_exp = np.where(has, f, 0).astype(np.int64)
    if zero_frac > 0:
        z = rng.random(count) < zero_frac
        mant[z] = 0
        exps = np.where(z, 0, exps)
        kind = np.where(z, APB_ZERO, kind).astype(np.uint8)
        rad_man = np.where(z, 0, rad_man).astype(np.uint32)
        rad_exp = np.where(z, 0, rad_exp)
    return BallArray(mant, exps, kind, rad_man, rad_exp)


# ------------------------------------------------------------------ configs

def config1_dots(batch: int = 65536, n: int = 100, p: int = 128, seed_salt: int = 0):
    """c1: batch x n term pairs, p-bit mantissas, e in U[-8,8]; dots with index
    >= batch/2 carry radius 2^-130|m| on every x_i and y_i."""
    rng = rng_for(1, seed_salt)
    half = batch // 2
    xs, ys = [], []
    for rad in (None, 130):
        cnt = (half if rad is None else batch - half) * n
        xs.append(random_balls(rng, cnt, p, e_lo=-8, e_hi=8, rad_k=rad))
        ys.append(random_balls(rng, cnt, p, e_lo=-8, e_hi=8, rad_k=rad))
    return xs[0].concat(xs[1]), ys[0].concat(ys[1])


def config2_matrices(n: int = 256, p: int = 128, seed_salt: int = 0):
    """c2: A, B n x n, e in U[-4,4], radii 2^-130|m|"""
    rng = rng_for(2, seed_salt)
    a = random_balls(rng, n * n, p, e_lo=-4, e_hi=4, rad_k=130)
    b = random_balls(rng, n * n, p, e_lo=-4, e_hi=4, rad_k=130)
    return a, b


def config3_matrices(n: int = 512, p: int = 256, seed_salt: int = 0):
    """c3: row i of A at exponent e_i, column j of B at f_j, e,f in U[-200,200];
    10% exact zeros; 5% of nonzero entries radius 2^-40|m|"""
    rng = rng_for(3, seed_salt)
    ei = rng.integers(-200, 200, size=n, endpoint=True, dtype=np.int64)
    fj = rng.integers(-200, 200, size=n, endpoint=True, dtype=np.int64)
    a = random_balls(rng, n * n, p, exps=np.repeat(ei, n), rad_k=40, rad_frac=0.05, zero_frac=0.10)
    b = random_balls(rng, n * n, p, exps=np.tile(fj, n), rad_k=40, rad_frac=0.05, zero_frac=0.10)
    return a, b


def config4_matrices(n: int = 1024, p: int = 512, seed_salt: int = 0):
    """c4: complex A, B; Re/Im independent, e in U[-16,16], radii 2^-515|m|"""
    rng = rng_for(4, seed_salt)
    parts = [random_balls(rng, n * n, p, e_lo=-16, e_hi=16, rad_k=515) for _ in range(4)]
    return parts  # are, aim, bre, bim


def config5_matrices(n: int = 2048, p: int = 128, seed_salt: int = 0):
    rng = rng_for(5, seed_salt + p)
    a = random_balls(rng, n * n, p, e_lo=-32, e_hi=32, rad_k=p + 2)
    b = random_balls(rng, n * n, p, e_lo=-32, e_hi=32, rad_k=p + 2)
    return a, b


def config5_dots(batch: int = 8192, n: int = 1000, p: int = 128, seed_salt: int = 0):
    rng = rng_for(50, seed_salt + p)
    x = random_balls(rng, batch * n, p, e_lo=-32, e_hi=32, rad_k=p + 2)
    y = random_balls(rng, batch * n, p, e_lo=-32, e_hi=32, rad_k=p + 2)
    return x, y


def edge_dots(rng: np.random.Generator, batch: int, n: int, max_limbs: int = 4,
              spread: int = 200, specials: bool = True, zero_rad_pct: int = 60):
    """Mixed-edge-case dot inputs in the spirit of random_dot_instance
    (src/bench.cpp:414-458): variable limb counts, exact zeros, radii below
    the midpoint, optional specials (NaN/inf/huge exponents -> Fallback)."""
    L = max_limbs
    cnt = batch * n

    def one(cnt):
        nl = rng.integers(1, L + 1, size=cnt)
        m = rng.integers(0, np.iinfo(np.uint64).max, size=(cnt, L), dtype=np.uint64, endpoint=True)
        for j in range(L):  # keep only the top nl limbs (top-aligned)
            m[:, j] = np.where(L - j <= nl, m[:, j], 0)
        m[:, L - 1] |= np.uint64(1 << 63)
        lowest = np.clip(L - nl, 0, L - 1)
        rows = np.arange(cnt)
        m[rows, lowest] = np.where(m[rows, lowest] == 0, np.uint64(1), m[rows, lowest])
        e = rng.integers(-spread, spread, size=cnt, endpoint=True, dtype=np.int64)
        neg = rng.integers(0, 2, size=cnt).astype(bool)
        kind = np.where(neg, APB_FINITE | APB_SIGN, APB_FINITE).astype(np.uint8)
        zero = rng.random(cnt) < 0.10
        m[zero] = 0
        e = np.where(zero, 0, e)
        kind = np.where(zero, APB_ZERO, kind).astype(np.uint8)
        has_rad = rng.random(cnt) >= zero_rad_pct / 100.0
        rb = (np.uint64(1 << 29) + rng.integers(0, 1 << 29, size=cnt).astype(np.uint64)).astype(np.uint32)
        rf = np.where(zero, rng.integers(-spread, spread, size=cnt), e - rng.integers(0, 120, size=cnt))
        rf = rf - rng.integers(0, 3, size=cnt)
        rad_man = np.where(has_rad, rb, 0).astype(np.uint32)
        rad_exp = np.where(has_rad, rf, 0).astype(np.int64)
        return BallArray(m, e, kind, rad_man, rad_exp)

    x, y = one(cnt), one(cnt)
    if specials:
        from .balls import APB_NAN, APB_PINF, APB_NINF, APB_RAD_INF
        sel = rng.random(cnt) < 0.002
        for arr in (x,):
            k = rng.integers(0, 4, size=cnt)
            arr.kind = np.where(sel & (k == 0), APB_NAN, arr.kind).astype(np.uint8)
            arr.kind = np.where(sel & (k == 1), APB_PINF, arr.kind).astype(np.uint8)
            arr.kind = np.where(sel & (k == 2), APB_NINF, arr.kind).astype(np.uint8)
            arr.mant[sel & (k <= 2)] = 0
            arr.exp = np.where(sel & (k <= 2), 0, arr.exp)
            huge = sel & (k == 3) & ((arr.kind & 7) == APB_FINITE)
            arr.exp = np.where(huge, np.int64(1 << 61), arr.exp)
            arr.rad_man = np.where(huge, 0, arr.rad_man).astype(np.uint32)
            sel2 = rng.random(cnt) < 0.001
            arr.rad_man = np.where(sel2, APB_RAD_INF, arr.rad_man).astype(np.uint32)
        # the reference reads an empty limb vector in mag_upper_from_apfloat(+-inf)
        # when the other factor carries a radius (src/ball.cpp:29-32 with
        # src/mag.cpp:147-153, assert compiled out): its output radius is
        # unspecified there, so parity inputs keep such partners exact.
        infx = ((x.kind & 7) == APB_PINF) | ((x.kind & 7) == APB_NINF)
        y.rad_man = np.where(infx, 0, y.rad_man).astype(np.uint32)
    return x, y
