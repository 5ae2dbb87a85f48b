"""Exponent statistics (stats1/stats2 + the device selection) against the
oracle's two-stage restatement (precsel.cpp:23-45,89-104 via exp_stats /
exp_stats_staged) on adversarial layouts at 2^21 components: magnitudes rising
or falling along memory across all 277 binades (blocks whose maxima are
hundreds of binades apart, subnormal and Inf binades included), runs at
unrelated scales, and arbitrary bit patterns (subnormals, +-0, Inf, NaN), over
targets that put the stage-2 threshold in the subnormal range, above every
element, or nowhere (no e_max); plus both operands of an AUTO dispatch in one
grid.  Bit-exact: every count, e_max and the decision line."""
import numpy as np
import pytest
import torch

import oracle as O
from paper_2303_08989_b200 import SelectionPolicy, make_config
from tests.golden.recipes import random_bits

pytestmark = pytest.mark.gpu


def _layout(kind: str, n: int, seed: int) -> np.ndarray:
    """n complex64 values (2n floats)."""
    rng = np.random.default_rng(seed)
    nf = 2 * n
    if kind == "bits":
        return random_bits(seed, nf).view(np.complex64)
    if kind in ("rising", "falling"):
        e = np.linspace(-149, 127, nf)
        if kind == "falling":
            e = e[::-1]
        e = np.floor(e).astype(np.int64)
        mant = rng.integers(0, 1 << 23, nf, dtype=np.uint32)
        biased = np.clip(e + 127, 0, 254).astype(np.uint32)
        sub = e < -126  # subnormal binades: a leading one at bit e + 149
        bitsv = np.where(sub, (np.uint32(1) << np.clip(e + 149, 0, 22).astype(np.uint32)) |
                         (mant & ((np.uint32(1) << np.clip(e + 149, 0, 22).astype(np.uint32)) - 1)),
                         (biased << 23) | mant)
        bitsv |= rng.integers(0, 2, nf, dtype=np.uint32) << 31
        x = bitsv.astype(np.uint32).view(np.float32)
    else:  # "blocks": runs of 3000 floats at unrelated scales, plus specials
        x = rng.standard_normal(nf).astype(np.float32)
        run = 3000
        scales = rng.integers(-140, 120, (nf + run - 1) // run)
        x *= np.repeat(np.ldexp(np.float32(1), scales).astype(np.float32), run)[:nf]
    x = x.copy()
    idx = rng.choice(nf, min(64, nf), replace=False)
    x[idx[:16]] = 0.0
    x[idx[16:24]] = -0.0
    x[idx[24:32]] = np.inf
    x[idx[32:40]] = np.nan
    x[idx[40:48]] = np.float32(1e-45)
    return x.view(np.complex64)


@pytest.mark.parametrize("kind", ["rising", "falling", "blocks", "bits"])
def test_stats_adversarial_layouts_match_oracle(handle, orc, dev, kind):
    host = _layout(kind, 1 << 20, 31)
    md = torch.from_numpy(host).to(dev).reshape(1, -1)
    hm = host.reshape(1, -1)
    for target in (14, 15, 17, 0, -14, 18, 40):
        assert handle.exp_stats(md, target).as_tuple() == \
            tuple(orc.exp_stats(hm, target).as_dict().values()), (kind, target)
        for t in (0.0, 0.3, 1.0):
            got = handle.exp_stats_staged(md, target, t).as_tuple()
            assert got == tuple(orc.exp_stats_staged(hm, target, t).as_dict().values()), (kind, target, t)


@pytest.mark.parametrize("n", [1, 5, 4097, 300001])
def test_stats_sizes_and_offsets(handle, orc, dev, n):
    # sizes around the float4 split and unaligned starts (the scalar tail)
    host = _layout("rising", n + 3, 7 + n)
    big = torch.from_numpy(host).to(dev).reshape(-1)
    for off in (0, 1, 3):
        sub = big[off:off + n].reshape(1, -1)
        want = host[off:off + n].reshape(1, -1)
        assert handle.exp_stats_staged(sub, 14, 0.0).as_tuple() == \
            tuple(orc.exp_stats_staged(want, 14, 0.0).as_dict().values()), (n, off)


@pytest.mark.parametrize("kinds", [("rising", "falling"), ("blocks", "bits"), ("falling", "blocks")])
def test_dispatch_decision_adversarial_operands(handle, orc, dev, kinds):
    # both operands in one statistics grid, then the device selection: statistics,
    # decision and log line equal to the reference restatement
    m, k, n = 512, 768, 640
    a_h = _layout(kinds[0], m * k, 3).reshape(m, k)
    b_h = _layout(kinds[1], k * n, 4).reshape(k, n)
    a_h = np.where(np.isfinite(a_h), a_h, np.complex64(0.5))  # finite: the GEMM runs
    b_h = np.where(np.isfinite(b_h), b_h, np.complex64(-0.25))
    for t, target in ((0.0, 14), (0.5, 14), (0.2, 15)):
        pol = SelectionPolicy(threshold_t=t, size_auto=256, size_tf32=256, target_max_exponent=target)
        _, res = handle.dispatch_cgemm(torch.from_numpy(a_h).to(dev), torch.from_numpy(b_h).to(dev),
                                       make_config(pol))
        rc, want = orc.dispatch_decision(a_h, b_h, O.make_config(threshold_t=t, size_auto=256,
                                                                  size_tf32=256, target=target))
        assert rc == 0
        assert res.line == want.line.decode(), (kinds, t, res.line, want.line)
        for s_dev, s_ref in ((res.stats_a, want.stats_a), (res.stats_b, want.stats_b)):
            assert (s_dev.n1, s_dev.n2, s_dev.n_nonzero, s_dev.n_total, s_dev.e_max) == \
                   (s_ref.n1, s_ref.n2, s_ref.n_nonzero, s_ref.n_total, s_ref.e_max), (kinds, t)
