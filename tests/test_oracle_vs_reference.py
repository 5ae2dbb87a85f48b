"""Live pin of the C restatement against the reference build (oracle/_ref) on
fresh random inputs.  Skipped where the reference could not be built."""
import numpy as np
import pytest

import oracle as O
from tests.conftest import bits
from tests.golden.recipes import SPECIALS, matrix_recipe, random_bits


def test_lowprec_random_bits(orc, ref):
    x = np.concatenate([np.array(SPECIALS, np.float32), random_bits(99, 200000)])
    for fmt in (0, 1):
        for rd in (0, 1):
            a, oa = orc.quantize_buf(x, fmt, rd)
            b, ob = ref.quantize_buf(x, fmt, rd)
            assert np.array_equal(bits(a), bits(b)) and oa == ob
        ha, la, oa = orc.split_buf(x, fmt)
        hb, lb, ob = ref.split_buf(x, fmt)
        assert np.array_equal(bits(ha), bits(hb)) and np.array_equal(bits(la), bits(lb)) and oa == ob
    for s in (-200, -64, -3, 0, 5, 40, 130, 5000):
        assert np.array_equal(bits(orc.scale_buf(x, s)), bits(ref.scale_buf(x, s)))
    for a, b in zip(x[:2000], x[2000:4000]):
        assert np.float32(orc.add_rz(a, b)).view(np.uint32) == np.float32(ref.add_rz(a, b)).view(np.uint32)


@pytest.mark.parametrize("recipe", ["uniform", "tiny20", "huge20", "type3", "subnormal", "sparse",
                                    "mixed40", "banded"])
def test_stats_random(orc, ref, recipe):
    for seed in range(5):
        m = matrix_recipe(recipe, 23 + seed, 31, 50 + seed)
        assert orc.exp_stats(m).as_dict() == ref.exp_stats(m).as_dict()
        for t in (0.0, 0.3, 1.0):
            so, sr = orc.exp_stats_staged(m, 14, t), ref.exp_stats_staged(m, 14, t)
            assert so.as_dict() == sr.as_dict()
            assert orc.matrix_tolerance(so, t) == ref.matrix_tolerance(sr, t)


def test_cgemm_random_shapes(orc, ref):
    g = np.random.default_rng(3)
    for it in range(6):
        m, n, k = (int(v) for v in g.integers(1, 40, 3))
        a = matrix_recipe("uniform", m, k, 900 + it)
        b = matrix_recipe("banded", k, n, 950 + it)
        for mode in O.MODES:
            for kt in (1, 16, 7):
                ca, _ = orc.cgemm(a, b, mode, kt)
                cb, _ = ref.cgemm(a, b, mode, kt)
                assert np.array_equal(bits(ca.view(np.float32)), bits(cb.view(np.float32)))


def test_dispatch_lines_random(orc, ref):
    for it, (ra, rb) in enumerate([("uniform", "type3"), ("tiny20", "banded"), ("huge20", "uniform"),
                                   ("sparse", "subnormal")]):
        a = matrix_recipe(ra, 40, 36, 11 + it)
        b = matrix_recipe(rb, 36, 44, 21 + it)
        for t in (0.0, 0.25, 0.9):
            cfg = O.make_config(threshold_t=t, size_auto=32, size_tf32=16)
            ro, co, reso = orc.dispatch_cgemm(a, b, cfg)
            rr, cr, resr = ref.dispatch_cgemm(a, b, cfg)
            assert ro == rr and reso.line == resr.line
            assert np.array_equal(bits(co.view(np.float32)), bits(cr.view(np.float32)))
