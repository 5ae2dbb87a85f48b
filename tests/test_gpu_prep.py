"""Bit-exact parity of the hot path's operand preparation (prep_a / prep_b, the
kernels every tensor-core dispatch runs) against the reference arithmetic:

    hi, lo = split_buf(scale_buf(x, s), fmt)        kernels_scalar.cpp:24-40,
                                                    lowprec.hpp:58-88

rearranged into the tensor-core layout: A' = A viewed as m x 2k (interleaved
re/im along K), B'^T = the 2n x 2k block expansion with row 2j = (Br, -Bi) and
row 2j+1 = (Bi, Br) per complex k, both K-major and zero padded to
kp = round_up(2k, 64).  Every case is checked in both operand layouts: the
B-expanded one above and the A-expanded one (tcec_set_operand_layout, used
when m < n): A'' row 2i = (Ar, -Ai), row 2i+1 = (Ai, Ar); B'' row j = (Br, Bi)
= column j of B.  The oracle (the C restatement, pinned to the reference
build) is the checker; the device planes come back through
tcec_debug_prep_layout.  Uncorrected (TC ablation) preparation is pinned
against quantize_buf(RN).
"""
import numpy as np
import pytest
import torch

import oracle as O
from tests.golden.recipes import SPECIALS, random_bits

pytestmark = pytest.mark.gpu

KIND = {"FP16TCEC": 0, "FP16TCEC_SCALED": 1, "TF32TCEC": 2}


def _to_fmt(v, fmt):
    """f32 values that are exact in the target format -> the device storage type."""
    return v.astype(np.float16) if fmt == 0 else v.astype(np.float32)


def _expected(orc, a, b, kind, sa, sb, corrected, xa=False):
    fmt = 1 if kind == 2 else 0
    m, k = a.shape
    n = b.shape[1]
    kp = ((2 * k + 63) // 64) * 64
    ovf = False
    bad = False

    def prep(x, s):
        nonlocal ovf, bad
        x = np.ascontiguousarray(x, np.float32).ravel()
        if kind == 1:  # scale_matrix runs (and checks) even for a zero shift
            x = orc.scale_buf(x, s)
            bad |= bool((~np.isfinite(x)).any())
        if corrected:
            hi, lo, o = orc.split_buf(x, fmt)
        else:
            hi, o = orc.quantize_buf(x, fmt, 0)
            lo = np.zeros_like(hi)
        ovf |= bool(o)
        return hi, lo

    ah, al = prep(a.view(np.float32), sa)
    bh, bl = prep(b.view(np.float32), sb)
    if xa:
        A_hi = np.zeros((2 * m, kp), np.float32)
        A_lo = np.zeros((2 * m, kp), np.float32)
        for src, dst in ((ah, A_hi), (al, A_lo)):
            s = src.reshape(m, k, 2)
            re, im = s[:, :, 0], s[:, :, 1]                     # m x k
            dst[0::2, 0:2 * k:2] = re
            dst[0::2, 1:2 * k:2] = -im
            dst[1::2, 0:2 * k:2] = im
            dst[1::2, 1:2 * k:2] = re
        B_hi = np.zeros((n, kp), np.float32)
        B_lo = np.zeros((n, kp), np.float32)
        for src, dst in ((bh, B_hi), (bl, B_lo)):
            dst[:, :2 * k] = src.reshape(k, n, 2).transpose(1, 0, 2).reshape(n, 2 * k)
        return [_to_fmt(p, fmt) for p in (A_hi, A_lo, B_hi, B_lo)], ovf, bad
    A_hi = np.zeros((m, kp), np.float32)
    A_lo = np.zeros((m, kp), np.float32)
    A_hi[:, :2 * k] = ah.reshape(m, 2 * k)
    A_lo[:, :2 * k] = al.reshape(m, 2 * k)

    B_hi = np.zeros((2 * n, kp), np.float32)
    B_lo = np.zeros((2 * n, kp), np.float32)
    for src, dst in ((bh, B_hi), (bl, B_lo)):
        s = src.reshape(k, n, 2)
        re, im = s[:, :, 0].T, s[:, :, 1].T                     # n x k
        dst[0::2, 0:2 * k:2] = re
        dst[0::2, 1:2 * k:2] = -im
        dst[1::2, 0:2 * k:2] = im
        dst[1::2, 1:2 * k:2] = re
    return [_to_fmt(p, fmt) for p in (A_hi, A_lo, B_hi, B_lo)], ovf, bad


def _same_bits(got, want):
    got = np.ascontiguousarray(got)
    want = np.ascontiguousarray(want)
    u = np.uint16 if got.dtype == np.float16 else np.uint32
    gn, wn = np.isnan(got), np.isnan(want)
    if not np.array_equal(gn, wn):
        return False
    return np.array_equal(got.view(u)[~gn], want.view(u)[~wn])


def _check(handle, orc, a, b, kind, sa=0, sb=0, corrected=True, check_bits=True):
    for xa in (False, True):
        _check_layout(handle, orc, a, b, kind, sa, sb, corrected, check_bits, xa)


def _check_layout(handle, orc, a, b, kind, sa, sb, corrected, check_bits, xa):
    dev = torch.device("cuda:0")
    ad = torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    bd = torch.from_numpy(np.ascontiguousarray(b)).to(dev)
    *planes, ovf, bad = handle.debug_prep(ad, bd, kind, sa, sb, corrected, xa=xa)
    want, wovf, wbad = _expected(orc, a, b, KIND[kind], sa, sb, corrected, xa)
    assert bad == wbad, ("ScaleOverflow flag", bad, wbad, xa)
    if bad:
        return  # the reference throws ScaleOverflow before splitting (precsel.cpp:54-57)
    assert ovf == wovf, ("overflow flag", ovf, wovf, xa)
    names = ("A_hi", "A_lo", "B'_hi", "B'_lo") if corrected else ("A_hi", None, "B'_hi", None)
    for name, g, w in zip(names, planes, want):
        if name is None:
            continue
        g = g.cpu().numpy()
        if check_bits:
            assert _same_bits(g, w), (name, "xa" if xa else "bx", kind, sa, sb, np.argwhere(
                g.view(np.uint16 if g.dtype == np.float16 else np.uint32)
                != w.view(np.uint16 if w.dtype == np.float16 else np.uint32))[:5])


def _c(x):
    x = np.ascontiguousarray(x, np.float32)
    return x.view(np.complex64)


def _uniform(seed, r, c):
    return O.Rng(seed).uniform_c32(r, c)


def _bits_matrix(seed, r, c, lo_exp=None, hi_exp=None):
    """Random f32 bit patterns (subnormals included), optionally limited to a
    binary exponent window so a shift keeps them finite."""
    x = random_bits(seed, 2 * r * c * 2)
    if lo_exp is not None:
        e = np.floor(np.log2(np.abs(x.astype(np.float64)) + 1e-300))
        x = x[(e >= lo_exp) & (e <= hi_exp) | (x == 0)]
        x = np.resize(x, 2 * r * c)
    return _c(x[:2 * r * c].reshape(r, 2 * c))


def _specials_matrix(r, c, seed=0):
    g = np.random.default_rng(seed)
    sp = np.array(SPECIALS, np.float32)
    x = np.concatenate([sp, -sp, random_bits(seed + 9, 2 * r * c)])
    x = x[g.permutation(len(x))][:2 * r * c]
    return _c(x.reshape(r, 2 * c))


@pytest.mark.parametrize("kind", ["FP16TCEC", "TF32TCEC"])
@pytest.mark.parametrize("shape", [(1, 1, 1), (3, 5, 7), (64, 64, 32), (130, 70, 33), (256, 96, 100),
                                   (17, 300, 200)])
def test_prep_uniform_bit_exact(handle, orc, kind, shape):
    m, n, k = shape
    _check(handle, orc, _uniform(m + 7, m, k), _uniform(n + 11, k, n), kind)


@pytest.mark.parametrize("kind", ["FP16TCEC", "TF32TCEC"])
@pytest.mark.parametrize("shape", [(40, 24, 36), (128, 64, 64), (5, 9, 3)])
def test_prep_random_bits_subnormals_saturation(handle, orc, kind, shape):
    """The whole f32 range: FP16/TF32 subnormals, rounding at the format
    boundary, saturation past the format maximum (overflow flag), +-0."""
    m, n, k = shape
    a = _bits_matrix(1 + m, m, k)
    b = _bits_matrix(2 + n, k, n)
    _check(handle, orc, a, b, kind)


@pytest.mark.parametrize("kind", ["FP16TCEC", "TF32TCEC"])
def test_prep_specials(handle, orc, kind):
    """Reference special values (test_kernels.cpp:20-42 family): 2^-14, 2^-24,
    2^-25 (tie to zero), 65504 / 65520 (saturation), TF32 maximum and past it,
    +-inf, +-0, f32 subnormals."""
    a = _specials_matrix(24, 20, seed=3)
    b = _specials_matrix(20, 16, seed=4)
    _check(handle, orc, a, b, kind)


def test_prep_nan_propagates(handle, orc):
    a = _uniform(5, 16, 16)
    a.view(np.float32)[3, 5] = np.nan
    b = _uniform(6, 16, 16)
    b.view(np.float32)[7, 2] = np.float32("nan")
    for kind in ("FP16TCEC", "TF32TCEC"):
        _check(handle, orc, a, b, kind)


@pytest.mark.parametrize("sa,sb", [(15, 15), (14, 15), (1, -1), (35, 35), (-7, 20), (127, 0),
                                   (-126, 3), (-149, 0), (-140, 30)])
def test_prep_scaled_fast_path(handle, orc, sa, sb):
    """FP16TCEC_SCALED with shifts whose 2^s is an f32 (the vectorised
    __fmul_rn path): one rounding of the exact product, as
    float(double(x) * 2^s)."""
    m, n, k = 48, 40, 36
    a = _bits_matrix(abs(10 + sa), m, k, lo_exp=-149, hi_exp=min(127, 127 - sa))
    b = _bits_matrix(abs(20 + sb), k, n, lo_exp=-149, hi_exp=min(127, 127 - sb))
    _check(handle, orc, a, b, "FP16TCEC_SCALED", sa, sb)


@pytest.mark.parametrize("sa,sb", [(150, 0), (-150, 140), (200, -170), (-163, 163), (1100, 0),
                                   (0, -300)])
def test_prep_scaled_double_path(handle, orc, sa, sb):
    """Shifts outside [-149, 127] take the double path; values chosen so the
    scaled operand stays finite, plus underflow to +-0 / subnormals."""
    m, n, k = 32, 24, 20

    def window(s):
        lo = max(-149, -149 - s)
        hi = min(127, 127 - s)
        return (lo, hi) if lo <= hi else (-149, 127)

    la, ha = window(sa)
    lb, hb = window(sb)
    a = _bits_matrix(30, m, k, lo_exp=la, hi_exp=ha)
    b = _bits_matrix(31, k, n, lo_exp=lb, hi_exp=hb)
    _check(handle, orc, a, b, "FP16TCEC_SCALED", sa, sb)


@pytest.mark.parametrize("sa,sb", [(200, 0), (0, 40), (130, 130)])
def test_prep_scale_overflow_flag(handle, orc, sa, sb):
    """A shift that pushes a component past the f32 range raises the
    ScaleOverflow flag exactly when the reference's scale_matrix would throw."""
    a = _bits_matrix(40, 16, 16)
    b = _bits_matrix(41, 16, 16)
    _check(handle, orc, a, b, "FP16TCEC_SCALED", sa, sb)


@pytest.mark.parametrize("kind", ["FP16TCEC", "TF32TCEC"])
def test_prep_uncorrected_matches_quantize(handle, orc, kind):
    """TC ablation (gemm_tc): hi = quantize_buf(x, fmt, RN); lo unused."""
    a = _bits_matrix(50, 33, 21)
    b = _bits_matrix(51, 21, 19)
    _check(handle, orc, a, b, kind, corrected=False)


def test_prep_large_ragged(handle, orc):
    """A larger ragged case through the vectorised paths (k not a multiple of
    the 64-element k-block; misaligned row starts)."""
    a = _uniform(77, 1000, 517)
    b = _uniform(78, 517, 333)
    a.view(np.float32)[::97, ::13] *= np.float32(2.0 ** -20)
    b.view(np.float32)[::89, ::7] *= np.float32(2.0 ** 12)
    for kind, s in (("FP16TCEC", (0, 0)), ("TF32TCEC", (0, 0)), ("FP16TCEC_SCALED", (15, 2))):
        _check(handle, orc, a, b, kind, *s)
