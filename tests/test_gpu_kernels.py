"""GPU parity of the HBM-bound kernels against the oracle: bit-exact quantize,
split, scale, add/sub, exponent statistics, and permute (reference
test_kernels.cpp / test_precsel.cpp / test_tensor.cpp:33-75)."""
import numpy as np
import pytest
import torch

import oracle as O
from paper_2303_08989_b200 import InvalidPermutation, ScaleOverflow
from tests.conftest import bits
from tests.golden.recipes import SPECIALS, matrix_recipe, random_bits

pytestmark = pytest.mark.gpu


def _x():
    return np.concatenate([np.array(SPECIALS, np.float32), random_bits(123, 1 << 20)])


@pytest.mark.parametrize("n", [1, 7, 8, 33, 1000, 1 << 20])
def test_quantize_split_bit_exact(handle, orc, dev, n):
    x = _x()[:n] if n <= 1 << 20 else _x()
    xd = torch.from_numpy(x).to(dev)
    for fmt in (0, 1):
        for rd in (0, 1):
            y, ov = handle.quantize_buf(xd, fmt, rd)
            yr, ovr = orc.quantize_buf(x, fmt, rd)
            assert np.array_equal(bits(y.cpu().numpy()), bits(yr)) and ov == ovr
        hi, lo, ov = handle.split_buf(xd, fmt)
        hr, lr, ovr = orc.split_buf(x, fmt)
        assert np.array_equal(bits(hi.cpu().numpy()), bits(hr))
        assert np.array_equal(bits(lo.cpu().numpy()), bits(lr))
        assert ov == ovr


def test_lowprec_golden_on_device(handle, golden, dev):
    g = golden("lowprec.npz")
    x = g["x"].view(np.float32)
    xd = torch.from_numpy(x.copy()).to(dev)
    for fmt in (0, 1):
        for rd in (0, 1):
            y, ov = handle.quantize_buf(xd, fmt, rd)
            assert np.array_equal(bits(y.cpu().numpy()), g[f"q{fmt}{rd}"])
            assert ov == bool(g[f"q{fmt}{rd}_ovf"][0])
        hi, lo, ov = handle.split_buf(xd, fmt)
        assert np.array_equal(bits(hi.cpu().numpy()), g[f"hi{fmt}"])
        assert np.array_equal(bits(lo.cpu().numpy()), g[f"lo{fmt}"])
    for s in (0, 1, -7, 34, -163, 163, 1100):
        assert np.array_equal(bits(handle.scale_buf(xd, s).cpu().numpy()), g[f"scale{s}"])


def test_add_sub_bit_exact(handle, dev):
    a = random_bits(1, 5000)
    b = random_bits(2, 5000)
    ad, bd = torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev)
    with np.errstate(all="ignore"):
        assert np.array_equal(bits(handle.add_buf(ad, bd).cpu().numpy()), bits(a + b))
        assert np.array_equal(bits(handle.sub_buf(ad, bd).cpu().numpy()), bits(a - b))


@pytest.mark.parametrize("recipe", ["uniform", "tiny20", "huge20", "banded", "type3", "zeros",
                                    "subnormal", "mixed40", "ones", "sparse"])
def test_exp_stats_bit_exact(handle, orc, dev, recipe):
    for (rows, cols, seed) in ((4, 4, 1), (37, 29, 2), (128, 96, 3), (1, 1, 4), (513, 257, 5)):
        m = matrix_recipe(recipe, rows, cols, seed)
        md = torch.from_numpy(m).to(dev)
        assert handle.exp_stats(md).as_tuple() == tuple(orc.exp_stats(m).as_dict().values())
        for t in (0.0, 0.1, 0.5, 0.95, 1.0):
            got = handle.exp_stats_staged(md, 14, t).as_tuple()
            assert got == tuple(orc.exp_stats_staged(m, 14, t).as_dict().values()), (recipe, t)


def test_exp_stats_unaligned_views(handle, orc, dev):
    m = matrix_recipe("type3", 61, 17, 9)
    big = torch.from_numpy(m).to(dev).reshape(-1)
    for off in (1, 3):
        sub = big[off:]
        host = m.reshape(-1)[off:]
        assert handle.exp_stats(sub.reshape(1, -1)).as_tuple() == tuple(
            orc.exp_stats(host.reshape(1, -1)).as_dict().values())


def test_exp_stats_invariances(handle, dev):
    # power-of-two invariance and a planted outlier (test_precsel.cpp:151-181)
    m = matrix_recipe("uniform", 64, 64, 405) * np.float32(2.0 ** -8)
    base = handle.exp_stats(torch.from_numpy(m).to(dev))
    for s in (-6, -1, 3, 10):
        st = handle.exp_stats(torch.from_numpy(m * np.float32(2.0 ** s)).to(dev))
        assert (st.n_nonzero, st.n2, st.e_max) == (base.n_nonzero, base.n2, base.e_max + s)
    band = matrix_recipe("banded", 16, 16, 406)
    before = handle.exp_stats(torch.from_numpy(band).to(dev))
    band[3, 7] = np.complex64(2.0 ** -60 + 0.5j)
    after = handle.exp_stats(torch.from_numpy(band).to(dev))
    assert after.n2 == before.n2 - 1


def test_scale_matrix_overflow_and_roundtrip(handle, dev):
    m = torch.from_numpy(matrix_recipe("uniform", 8, 8, 408)).to(dev)
    up = handle.scale_matrix(m, 17)
    assert torch.equal(handle.scale_matrix(up, -17), m)
    with pytest.raises(ScaleOverflow):
        handle.scale_matrix(torch.ones(2, 2, dtype=torch.complex64, device=dev), 128)
    ones = torch.ones(3, 3, dtype=torch.complex64, device=dev) * (1 + 1j)
    handle.descale_output_inplace(ones, 14, 34)
    assert torch.all(ones.real == 2.0 ** -48) and torch.all(ones.imag == 2.0 ** -48)


def test_permute_bit_exact(handle, golden, dev):
    for case, d in golden("permute.json").items():
        t = matrix_recipe("uniform", 1, int(np.prod(d["dims"])), 700 + int(case)).reshape(d["dims"])
        out = handle.permute(torch.from_numpy(t).to(dev), d["axis"]).cpu().numpy()
        assert bits(out.reshape(-1).view(np.float32)).tolist() == d["out"]


def test_permute_high_rank_dim2(handle, dev):
    g = np.random.default_rng(4)
    for r in (8, 16, 22):
        t = torch.randn(*([2] * r), dtype=torch.complex64, device=dev)
        axis = [int(v) for v in g.permutation(r)]
        assert torch.equal(handle.permute(t, axis), t.permute(*axis).contiguous())


@pytest.mark.parametrize("rank,axis", [
    (22, [20, 21, 0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15, 16, 17, 18, 19]),
    (22, [9, 3, 14, 0, 1, 2, 4, 5, 6, 7, 8, 10, 11, 12, 13, 15, 16, 17, 18, 19, 20, 21]),
    (20, [14, 2, 0, 1, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 15, 16, 17, 18, 19]),
    (12, [11, 10, 9, 8, 7, 0, 1, 2, 3, 4, 5, 6]),
    (24, [1, 12, 5, 23, 18, 14, 0, 2, 3, 4, 6, 7, 8, 9, 10, 11, 13, 15, 16, 17, 19, 20, 21, 22]),
    (21, [0, 1, 2, 3, 4, 5, 6, 8, 9, 10, 11, 12, 13, 14, 15, 7, 16, 17, 18, 19, 20]),
])
def test_permute_run_copy(handle, dev, rank, axis):
    """Permutations that keep >= 32 innermost elements in place (a few outer
    axes moved -- the common TTGT case of sliced circuit intermediates) take
    the run-copy kernel; bit-exact, including runs of exactly 32."""
    t = torch.randn(*([2] * rank), dtype=torch.complex64, device=dev)
    assert torch.equal(handle.permute(t, axis), t.permute(*axis).contiguous())


def test_permute_errors(handle, dev):
    t = torch.zeros(2, 3, 4, dtype=torch.complex64, device=dev)
    with pytest.raises(InvalidPermutation):
        handle.permute(t, [0, 1])
    with pytest.raises(InvalidPermutation):
        handle.permute(t, [0, 1, 1])


@pytest.mark.parametrize("dims", [(2,) * 14, (2,) * 20, (4, 8, 16, 32), (128, 3, 256), (96, 64),
                                  (2, 64, 2, 64), (33, 70, 5), (2,) * 25, (1024, 2, 512),
                                  (8, 2, 1024, 4), (2, 2, 2, 2, 2, 2, 2, 2, 2, 2, 4)])
def test_permute_tiled_and_gather_paths(handle, dev, dims):
    """Random permutations of shapes that exercise the bit-permutation plan
    (power-of-two extents), the shared-memory tiled plan (axes split at 32) and
    the gather fallback; bit-exact."""
    g = np.random.default_rng(len(dims) * 7 + dims[0])
    t = torch.randn(*dims, dtype=torch.complex64, device=dev)
    for _ in range(4):
        axis = [int(v) for v in g.permutation(len(dims))]
        assert torch.equal(handle.permute(t, axis), t.permute(*axis).contiguous()), axis
