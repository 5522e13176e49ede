"""CPU model of the int8 digit splitting behind csrc/ozaki.cu (no GPU): the
same scaling, digit extraction, product selection (p + q <= 7) and integer
recombination in numpy / Python integers, checked against exact rational
arithmetic.  Pins the error claim of DESIGN.md section 3 item 8: per k-term
below 2^-53 rowmax(A) colmax(B), digits in [-64, 64], int32 accumulators."""
from fractions import Fraction

import numpy as np

S = 8  # slices


def split(x, axis_scale):
    """x (2-D float64) scaled by 2^(6 - e) per row (axis_scale: e per row, shape (rows, 1)) ->
    digits[s] (int64) with x ~= 2^(e - 6) sum_s digits[s] 2^(-7 s)."""
    t = x * np.exp2(6.0 - axis_scale)
    digits = []
    for _ in range(S):
        d = np.rint(t)
        digits.append(d.astype(np.int64))
        t = (t - d) * 128.0
    return digits


def exponent(mx):
    e = np.zeros_like(mx)
    nz = mx > 0
    e[nz] = np.floor(np.log2(mx[nz])) + 1
    return e


def ozaki_real(a, b):
    """a (m x k), b (k x n) real -> a @ b by the slice scheme, with the accumulator maxima."""
    ea = exponent(np.abs(a).max(axis=1, keepdims=True))
    eb = exponent(np.abs(b).max(axis=0, keepdims=True))
    da = split(a, ea)
    db = [d.T for d in split(b.T.copy(), eb.T.copy())]
    acc = [sum(da[p] @ db[d - p] for p in range(d + 1)) for d in range(S)]
    hi = sum(acc[d] << (7 * (3 - d)) for d in range(4))
    lo = sum(acc[d] << (7 * (7 - d)) for d in range(4, 8))
    v = hi.astype(np.float64) * 2.0 ** -21 + lo.astype(np.float64) * 2.0 ** -49
    out = v * np.exp2(ea - 6.0) * np.exp2(eb - 6.0)
    return out, da, db, acc


def exact(a, b):
    m, k = a.shape
    n = b.shape[1]
    fa = [[Fraction(float(x)) for x in row] for row in a]
    fb = [[Fraction(float(x)) for x in row] for row in b]
    return [[sum(fa[i][t] * fb[t][j] for t in range(k)) for j in range(n)] for i in range(m)]


def test_digits_are_int8_and_reconstruct():
    rng = np.random.default_rng(0)
    a = rng.standard_normal((16, 48)) * 10.0 ** rng.uniform(-20, 20, (16, 1))
    ea = exponent(np.abs(a).max(axis=1, keepdims=True))
    da = split(a, ea)
    assert all(np.abs(d).max() <= 64 for d in da)
    rec = sum(d.astype(np.float64) * 2.0 ** (-7 * s) for s, d in enumerate(da)) * np.exp2(ea - 6.0)
    # 6 + 7 * 7 = 55 bits below the row maximum
    assert (np.abs(rec - a) <= 2.0 ** -55 * np.exp2(ea)).all()


def test_error_bound_against_exact_arithmetic():
    rng = np.random.default_rng(1)
    m, k, n = 6, 64, 5
    a = rng.standard_normal((m, k)) * 10.0 ** rng.uniform(-8, 8, (m, 1))
    b = rng.standard_normal((k, n)) * 10.0 ** rng.uniform(-8, 8, (1, n))
    got, da, db, acc = ozaki_real(a, b)
    ref = exact(a, b)
    ra = np.abs(a).max(axis=1)
    cb = np.abs(b).max(axis=0)
    for i in range(m):
        for j in range(n):
            err = abs(Fraction(float(got[i, j])) - ref[i][j])
            # per k-term below 2^-53 rowmax colmax (4x: the scales round the maxima up to powers of two),
            # plus the final FP64 roundings of the recombination
            bound = Fraction(4 * k) * Fraction(2) ** -53 * Fraction(float(ra[i])) * Fraction(float(cb[j]))
            assert err <= bound + abs(ref[i][j]) * Fraction(2) ** -51, (i, j, float(err), float(bound))


def test_accumulators_fit_int32_at_the_largest_k():
    """|digit| <= 64, at most 8 products per weight, K' = 2 k = 8192 bytes (K = 4096, the entry's limit)."""
    assert 8 * 8192 * 64 * 64 < 2 ** 31
    # and the two int64 recombinations cannot overflow
    assert (8 * 8192 * 64 * 64) * (2 ** 21 + 2 ** 14 + 2 ** 7 + 1) < 2 ** 63


def test_complex_embedding():
    """[Re A | Im A] times the rows [Re b; -Im b] and [Im b; Re b] gives (re, im) of A b."""
    rng = np.random.default_rng(2)
    a = rng.standard_normal((4, 8)) + 1j * rng.standard_normal((4, 8))
    b = rng.standard_normal((8, 3)) + 1j * rng.standard_normal((8, 3))
    ap = np.concatenate([a.real, a.imag], axis=1)
    rows = np.empty((6, 16))
    rows[0::2] = np.concatenate([b.real, -b.imag], axis=0).T
    rows[1::2] = np.concatenate([b.imag, b.real], axis=0).T
    out, *_ = ozaki_real(ap, rows.T.copy())
    c = a @ b
    assert np.allclose(out[:, 0::2], c.real, rtol=0, atol=1e-13) and np.allclose(out[:, 1::2], c.imag, rtol=0, atol=1e-13)
