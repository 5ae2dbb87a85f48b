"""GPU CGEMM parity (reference test_gemm.cpp / test_cgemm.cpp).

FP32_REF and FP64_ORACLE tiers are bit-identical to the reference schedule.
The tensor-core modes (tcgen05) accumulate in hardware order, so they are
checked against the f64 oracle with the reference's own acceptance bar:
    rel_err(TCEC) <= 4 * rel_err(FP32_REF on CPU)  and  <= 5e-6   (test_cgemm.cpp:64-66)
    rel_err(TC)   >= 10 * rel_err(TCEC)                             (test_gemm.cpp:98-101)
plus size-independent properties at full benchmark sizes.
"""
import numpy as np
import pytest
import torch

import oracle as O
from paper_2303_08989_b200 import InvalidArgument, SelectionPolicy, ShapeMismatch, make_config
from tests.conftest import bits
from tests.golden.recipes import matrix_recipe

pytestmark = pytest.mark.gpu

TOL_FACTOR = 4.0    # TCEC vs CPU FP32_REF error (test_cgemm.cpp:64-66)
TOL_ABS = 5e-6


def relerr(c, ref):
    c = np.asarray(c, dtype=np.complex128)
    return float(np.linalg.norm(c - ref) / np.linalg.norm(ref))


SHAPES = [(1, 1, 1), (3, 5, 7), (8, 32, 16), (13, 37, 65), (16, 48, 33), (64, 64, 64),
          (100, 1, 50), (1, 200, 3), (129, 65, 200), (300, 257, 31)]


@pytest.mark.parametrize("shape", SHAPES)
def test_fp32_ref_and_fp64_tiers_bit_exact(handle, orc, dev, shape):
    m, n, k = shape
    a = matrix_recipe("uniform", m, k, 1000 + m)
    b = matrix_recipe("uniform", k, n, 2000 + n)
    ad, bd = torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev)
    for mode in ("FP32_REF", "FP64_ORACLE"):
        c, _ = handle.cgemm(ad, bd, mode)
        cr, _ = orc.cgemm(a, b, mode)
        assert np.array_equal(bits(c.cpu().numpy().view(np.float32)), bits(cr.view(np.float32))), mode


def test_fp32_ref_golden(handle, golden, dev):
    g = golden("cgemm.npz")
    for (m, n, k) in SHAPES[:8]:
        a = matrix_recipe("uniform", m, k, 1000 + m)
        b = matrix_recipe("uniform", k, n, 2000 + n)
        c, _ = handle.cgemm(torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev), "FP32_REF")
        assert np.array_equal(bits(c.cpu().numpy().view(np.float32)), g[f"{m}x{n}x{k}:FP32_REF"])


@pytest.mark.parametrize("n", [256, 512, 1024, 2048])
def test_tcec_accuracy_uniform(handle, orc, dev, n):
    r = O.Rng(7 + n)
    a, b = r.uniform_c32(n, n), r.uniform_c32(n, n)
    ref = orc.cgemm_oracle(a, b)
    err_ref = relerr(orc.cgemm(a, b, "FP32_REF")[0], ref) if n <= 1024 else None
    ad, bd = torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev)
    errs = {}
    for mode in ("FP16TCEC", "TF32TCEC", "FP16TC", "TF32TC"):
        c, ovf = handle.cgemm(ad, bd, mode)
        assert not ovf
        errs[mode] = relerr(c.cpu().numpy(), ref)
    for mode in ("FP16TCEC", "TF32TCEC"):
        assert 1e-8 <= errs[mode] <= TOL_ABS, (mode, errs)
        if err_ref is not None:
            assert errs[mode] <= TOL_FACTOR * err_ref, (mode, errs, err_ref)
    assert errs["FP16TC"] >= 10 * errs["FP16TCEC"]
    assert errs["TF32TC"] >= 10 * errs["TF32TCEC"]


@pytest.mark.parametrize("shape", [(1, 1, 1), (3, 5, 7), (13, 37, 65), (129, 65, 200),
                                   (300, 257, 31), (1000, 7, 333), (5, 1100, 77), (130, 130, 1100)])
def test_tcec_ragged_shapes(handle, orc, dev, shape):
    m, n, k = shape
    a = matrix_recipe("uniform", m, k, 31 + m)
    b = matrix_recipe("uniform", k, n, 37 + n)
    ref = orc.cgemm_oracle(a, b)
    err_ref = relerr(orc.cgemm(a, b, "FP32_REF")[0], ref)
    ad, bd = torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev)
    for mode in ("FP16TCEC", "TF32TCEC"):
        c, _ = handle.cgemm(ad, bd, mode)
        e = relerr(c.cpu().numpy(), ref)
        assert e <= max(TOL_FACTOR * err_ref, 2e-7), (mode, e, err_ref)


@pytest.mark.parametrize("variant", ["single", "pair", "wide", "wide_persistent", "wide_mc", "pair_persistent"])
@pytest.mark.parametrize("shape", [(3, 5, 7), (129, 65, 200), (300, 257, 31), (513, 385, 129),
                                   (130, 130, 1100), (600, 300, 2100)])
def test_tcec_kernel_variants(handle, orc, dev, variant, shape):
    """Every tcgen05 kernel variant (128x128 single CTA, 256x128 and 256x256
    CTA pairs) meets the reference bar on ragged shapes; the TC ablation
    (no correction products) is >= 10x worse."""
    m, n, k = shape
    a = matrix_recipe("uniform", m, k, 41 + m)
    b = matrix_recipe("uniform", k, n, 43 + n)
    ref = orc.cgemm_oracle(a, b)
    err_ref = relerr(orc.cgemm(a, b, "FP32_REF")[0], ref)
    ad, bd = torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev)
    handle.set_gemm_variant(variant)
    try:
        errs = {}
        for mode in ("FP16TCEC", "TF32TCEC", "FP16TC"):
            c, _ = handle.cgemm(ad, bd, mode)
            errs[mode] = relerr(c.cpu().numpy(), ref)
    finally:
        handle.set_gemm_variant("auto")
    for mode in ("FP16TCEC", "TF32TCEC"):
        assert errs[mode] <= max(TOL_FACTOR * err_ref, 2e-7), (mode, errs, err_ref)
    if k >= 64:
        assert errs["FP16TC"] >= 10 * errs["FP16TCEC"], errs


@pytest.mark.parametrize("variant", ["single", "wide", "wide_persistent", "wide_mc", "pair_persistent"])
def test_tcec_all_positive_long_k(handle, orc, dev, variant):
    """All-positive operands make tensor-core truncation a systematic bias;
    the per-k-block RN flush keeps TCEC within the reference bar."""
    m, n, k = 256, 160, 4000
    rng = np.random.default_rng(5)
    a = (rng.random((m, k)) + 1j * rng.random((m, k))).astype(np.complex64)
    b = (rng.random((k, n)) + 1j * rng.random((k, n))).astype(np.complex64)
    ref = orc.cgemm_oracle(a, b)
    err_ref = relerr(orc.cgemm(a, b, "FP32_REF")[0], ref)
    handle.set_gemm_variant(variant)
    try:
        for mode in ("FP16TCEC", "TF32TCEC"):
            c, _ = handle.cgemm(torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev), mode)
            e = relerr(c.cpu().numpy(), ref)
            assert e <= TOL_FACTOR * err_ref, (variant, mode, e, err_ref)
    finally:
        handle.set_gemm_variant("auto")


def test_exact_small_value_matrices_all_modes(handle, dev):
    # test_gemm.cpp:166-181: {0, +-1/2, +-1} products are exact in every mode
    g = np.random.default_rng(31)
    vals = np.array([0.0, 0.5, -0.5, 1.0, -1.0], np.float32)
    for _ in range(20):
        a = (vals[g.integers(0, 5, (6, 9))] + 1j * vals[g.integers(0, 5, (6, 9))]).astype(np.complex64)
        b = (vals[g.integers(0, 5, (9, 5))] + 1j * vals[g.integers(0, 5, (9, 5))]).astype(np.complex64)
        want = a.astype(np.complex128) @ b.astype(np.complex128)
        ad, bd = torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev)
        for mode in ("FP32_REF", "FP64_ORACLE", "TF32TC", "FP16TC", "TF32TCEC", "FP16TCEC"):
            c, _ = handle.cgemm(ad, bd, mode)
            assert np.array_equal(c.cpu().numpy().astype(np.complex128), want), mode


def test_identity_operand_exact(handle, dev):
    # B entries exact in 11 significand bits (test_gemm.cpp:43-60, :147-164)
    g = np.random.default_rng(5)
    bv = (g.integers(-1024, 1025, (48, 40, 2)).astype(np.float32) / 1024).view(np.complex64)[..., 0]
    b = torch.from_numpy(np.ascontiguousarray(bv)).to(dev)
    eye = torch.eye(48, dtype=torch.complex64, device=dev)
    for mode in ("FP32_REF", "FP16TCEC", "TF32TCEC"):
        c, _ = handle.cgemm(eye, b, mode)
        assert torch.equal(c, b), mode


def test_power_of_two_scaling_commutes(handle, dev):
    # test_gemm.cpp:129-145 on the device: scaling A by 2^s scales C by 2^s exactly
    a = matrix_recipe("banded", 96, 80, 23)
    b = matrix_recipe("banded", 80, 112, 24)
    ad, bd = torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev)
    for mode in ("FP32_REF", "FP16TCEC", "TF32TCEC", "FP16TC", "TF32TC"):
        c, _ = handle.cgemm(ad, bd, mode)
        for s in (-3, -1, 1, 2, 5):
            cs, _ = handle.cgemm(ad * (2.0 ** s), bd, mode)
            assert torch.equal(cs, c * (2.0 ** s)), (mode, s)


def test_determinism(handle, dev):
    a = torch.from_numpy(matrix_recipe("uniform", 300, 200, 17)).to(dev)
    b = torch.from_numpy(matrix_recipe("uniform", 200, 260, 18)).to(dev)
    for mode in ("FP32_REF", "FP64_ORACLE", "TF32TC", "FP16TC", "TF32TCEC", "FP16TCEC"):
        c1, _ = handle.cgemm(a, b, mode)
        c2, _ = handle.cgemm(a, b, mode)
        assert torch.equal(c1, c2), mode


def test_flush_interval_is_accuracy_relevant(handle, orc, dev):
    """Without the RN flush the tensor-core main term truncates (error grows
    with k); the flush restores FP32-level accuracy."""
    r = O.Rng(99)
    a, b = r.uniform_c32(128, 4096), r.uniform_c32(4096, 128)
    ref = orc.cgemm_oracle(a, b)
    ad, bd = torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev)
    keep = handle.flush_kblocks
    try:
        handle.flush_kblocks = 0
        e0 = relerr(handle.cgemm(ad, bd, "FP16TCEC")[0].cpu().numpy(), ref)
        handle.flush_kblocks = keep
        e4 = relerr(handle.cgemm(ad, bd, "FP16TCEC")[0].cpu().numpy(), ref)
    finally:
        handle.flush_kblocks = keep
    assert e4 < e0 / 2


def test_overflow_flag(handle, dev):
    a = torch.full((4, 4), 70000.0 + 0j, dtype=torch.complex64, device=dev)
    b = torch.ones(4, 4, dtype=torch.complex64, device=dev)
    assert handle.cgemm(a, b, "FP16TCEC")[1]
    assert not handle.cgemm(a, b, "TF32TCEC")[1]


def test_shape_and_tiling_errors(handle, dev):
    a = torch.zeros(2, 3, dtype=torch.complex64, device=dev)
    b = torch.zeros(2, 2, dtype=torch.complex64, device=dev)
    with pytest.raises(ShapeMismatch):
        handle.cgemm(a, b, "FP32_REF")
    sq = torch.zeros(4, 4, dtype=torch.complex64, device=dev)
    with pytest.raises(InvalidArgument):
        handle.cgemm(sq, sq, "FP16TCEC", k_tile=0)
    handle.cgemm(sq, sq, "FP32_REF", k_tile=0)  # the FP32 tier takes no tiling (gemm.cpp:60-66)


def test_batched_reports_index(handle, dev):
    ok = (torch.zeros(4, 4, dtype=torch.complex64, device=dev),) * 2
    bad = (torch.zeros(4, 5, dtype=torch.complex64, device=dev),
           torch.zeros(4, 4, dtype=torch.complex64, device=dev))
    assert handle.cgemm_batched([], "FP32_REF") == []
    with pytest.raises(ShapeMismatch, match="batch entry 1"):
        handle.cgemm_batched([ok, bad], "FP32_REF")


@pytest.mark.slow
@pytest.mark.parametrize("n", [4096, 8192])
def test_tcec_full_size_row_sampled(handle, dev, n):
    """Benchmark sizes: rows sampled against an f64 product of those rows."""
    ah = (np.random.default_rng(n).uniform(-1, 1, (n, n, 2)).astype(np.float32)).view(np.complex64)[..., 0]
    bh = (np.random.default_rng(n + 1).uniform(-1, 1, (n, n, 2)).astype(np.float32)).view(np.complex64)[..., 0]
    ad, bd = torch.from_numpy(ah).to(dev), torch.from_numpy(bh).to(dev)
    rows = np.random.default_rng(3).choice(n, 16, replace=False)
    ref = ah[rows].astype(np.complex128) @ bh.astype(np.complex128)
    for mode in ("FP16TCEC", "TF32TCEC"):
        c, _ = handle.cgemm(ad, bd, mode)
        e = relerr(c[torch.from_numpy(rows).to(dev)].cpu().numpy(), ref)
        assert e <= 2e-6, (mode, e)


@pytest.mark.parametrize("shape", [(1 << 17, 2, 2), (2, 1 << 17, 2), (2, 2, 1 << 17),
                                   (70000, 3, 1), (3, 1, 70000), (1, 70000, 5)])
def test_extreme_aspect_shapes(handle, orc, dev, shape):
    """(2, 2^N, 2)-family and tall/long operands: the grid
    mappings must not hit the 65535 grid.y limit; FP32 tier bit-exact, TCEC
    within tolerance."""
    m, n, k = shape
    a = matrix_recipe("uniform", m, k, 5)
    b = matrix_recipe("uniform", k, n, 6)
    ad, bd = torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev)
    c, _ = handle.cgemm(ad, bd, "FP32_REF")
    cr, _ = orc.cgemm(a, b, "FP32_REF")
    assert np.array_equal(bits(c.cpu().numpy().view(np.float32)), bits(cr.view(np.float32)))
    c64, _ = handle.cgemm(ad, bd, "FP64_ORACLE")
    assert np.array_equal(bits(c64.cpu().numpy().view(np.float32)),
                          bits(orc.cgemm(a, b, "FP64_ORACLE")[0].view(np.float32)))
    ref = orc.cgemm_oracle(a, b)
    err_ref = relerr(cr, ref)
    for mode in ("FP16TCEC", "TF32TCEC"):
        cm, _ = handle.cgemm(ad, bd, mode)
        assert relerr(cm.cpu().numpy(), ref) <= max(TOL_FACTOR * err_ref, 3e-7), mode


@pytest.mark.parametrize("shape", [(1, 1, 300000), (2, 1, 70000), (3, 2, 50000), (1, 5, 4097), (64, 64, 2048),
                                   (7, 1, 1025), (100, 50, 5000), (256, 64, 4099), (33, 70, 1500)])
def test_long_k_kernels_bit_exact(handle, orc, dev, shape):
    """Few outputs, long k (the dot products of deep circuits): the warp-per-
    output kernels keep the reference's sequential chain order -> bit-exact."""
    m, n, k = shape
    a = matrix_recipe("uniform", m, k, 8)
    b = matrix_recipe("uniform", k, n, 9)
    ad, bd = torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev)
    for mode in ("FP32_REF", "FP64_ORACLE"):
        c, _ = handle.cgemm(ad, bd, mode)
        cr, _ = orc.cgemm(a, b, mode)
        assert np.array_equal(bits(c.cpu().numpy().view(np.float32)), bits(cr.view(np.float32))), mode


@pytest.mark.parametrize("shape", [(2, 4096, 2), (3, 5000, 7), (16, 8192, 32), (9, 4100, 1),
                                   (5000, 9, 31), (8192, 16, 1), (4096, 2, 2), (4097, 5, 17),
                                   (32, 5000, 8), (20, 4200, 100), (5000, 32, 128), (17, 4096, 64),
                                   (4100, 8, 8), (6000, 3, 24), (4133, 7, 9), (4096, 4, 16), (4111, 2, 40),
                                   # cp.async-staged column kernel (MX 8 / 16, k >= 8): ragged n, k % 8 != 0,
                                   # rows below MX, and a persistent walk over many 256-column chunks
                                   (8, 4099, 13), (6, 10001, 64), (12, 4500, 128), (16, 300001, 72),
                                   (5, 200000, 8), (31, 9000, 17)])
def test_skinny_kernels_bit_exact(handle, orc, dev, shape):
    """Irregular skinny shapes (k <= 128, one outer dim <= 32: PAPER.md:346-352)
    take the thread-per-column / thread-per-row kernels; the chains keep the
    reference order -> FP32_REF and FP64_ORACLE bit-exact."""
    m, n, k = shape
    a = matrix_recipe("uniform", m, k, 18 + m)
    b = matrix_recipe("uniform", k, n, 19 + n)
    ad, bd = torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev)
    for mode in ("FP32_REF", "FP64_ORACLE"):
        c, _ = handle.cgemm(ad, bd, mode)
        cr, _ = orc.cgemm(a, b, mode)
        assert np.array_equal(bits(c.cpu().numpy().view(np.float32)), bits(cr.view(np.float32))), mode


@pytest.mark.parametrize("shape", [(200, 150, 9000), (512, 512, 4096), (130, 70, 20000), (300, 260, 9000)])
@pytest.mark.parametrize("variant", ["single", "wide", "auto"])
def test_split_k_few_tiles_long_k(handle, orc, dev, shape, variant):
    """Few 128x128 tiles and a long K run split-K (partials summed in split
    order, descaled once): still within the reference bar for every TCEC
    mode, the descaled FP16TCEC_SCALED path included."""
    m, n, k = shape
    a = matrix_recipe("uniform", m, k, 61 + m)
    b = matrix_recipe("uniform", k, n, 67 + n)
    ref = orc.cgemm_oracle(a, b)
    err_ref = relerr(orc.cgemm(a, b, "FP32_REF")[0], ref)
    ad, bd = torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev)
    handle.set_gemm_variant(variant)
    try:
        for mode in ("FP16TCEC", "TF32TCEC"):
            c, _ = handle.cgemm(ad, bd, mode)
            assert relerr(c.cpu().numpy(), ref) <= TOL_FACTOR * err_ref, mode
        c, res = handle.dispatch_cgemm(ad * 2.0 ** -20, bd, SelectionPolicy(size_auto=64, size_tf32=32))
        assert "FP16TCEC_SCALED" in res.line
        assert relerr(c.cpu().numpy() * 2.0 ** 20, ref) <= TOL_FACTOR * err_ref
    finally:
        handle.set_gemm_variant("auto")


@pytest.mark.parametrize("shape", [(512, 256, 64), (512, 300, 100), (1024, 1000, 333), (2048, 512, 1000),
                                   (768, 640, 129), (512, 512, 9000), (4096, 2048, 512)])
@pytest.mark.parametrize("mode", ["FP16TCEC", "TF32TCEC", "AUTO", "SCALED"])
def test_multicast_clusters_bit_identical_to_pairs(handle, dev, shape, mode):
    """Clusters of two CTA pairs sharing B' tiles by TMA multicast run the same
    MMA sequence on the same operand bits as the single-pair wide kernel, so C
    is bit-identical -- odd tile counts (fallback), split-K (512^2 x 9000),
    the device-decided format (AUTO) and the scaled kind included."""
    m, n, k = shape
    a = matrix_recipe("uniform", m, k, 7 + m)
    b = matrix_recipe("uniform", k, n, 9 + n)
    if mode == "SCALED":
        a = (a * np.float32(2.0 ** -20)).astype(np.complex64)
    ad, bd = torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev)
    if mode in ("AUTO", "SCALED"):
        cfg = make_config(SelectionPolicy(size_auto=32, size_tf32=16))
    else:
        cfg = make_config(force=mode)
    outs, lines = {}, {}
    for variant in ("wide", "wide_mc"):
        handle.set_gemm_variant(variant)
        try:
            c, res = handle.dispatch_cgemm(ad, bd, cfg)
            outs[variant] = c.cpu().numpy()
            lines[variant] = res.line
        finally:
            handle.set_gemm_variant("auto")
    assert lines["wide"] == lines["wide_mc"]
    assert np.array_equal(outs["wide"].view(np.uint32), outs["wide_mc"].view(np.uint32)), lines["wide"]


@pytest.mark.parametrize("variant", ["auto", "single", "wide", "wide_persistent", "wide_mc", "pair_persistent"])
@pytest.mark.parametrize("shape", [(3, 5, 7), (64, 1000, 33), (129, 65, 200), (130, 600, 1100),
                                   (256, 4096, 64), (200, 150, 9000), (512, 2048, 512), (1, 300, 40)])
def test_operand_layouts(handle, orc, dev, variant, shape):
    """Both operand layouts -- the complex block expansion on B (B' = [[Br, Bi],
    [-Bi, Br]]) or on A (A'' rows (Ar, -Ai) / (Ai, Ar), C rows interleaved by
    the epilogue) -- meet the reference bar in every kernel variant, for the
    host-known kinds, the device-decided format and the descaled scaled kind;
    split-K (long k) and the persistent small-k kernel included."""
    m, n, k = shape
    a = matrix_recipe("uniform", m, k, 71 + m)
    b = matrix_recipe("uniform", k, n, 73 + n)
    ref = orc.cgemm_oracle(a, b)
    err_ref = relerr(orc.cgemm(a, b, "FP32_REF")[0], ref)
    ad, bd = torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev)
    handle.set_gemm_variant(variant)
    try:
        for layout in ("a", "b"):
            handle.set_operand_layout(layout)
            for mode in ("FP16TCEC", "TF32TCEC"):
                c, _ = handle.cgemm(ad, bd, mode)
                e = relerr(c.cpu().numpy(), ref)
                assert e <= max(TOL_FACTOR * err_ref, 2e-7), (layout, mode, e, err_ref)
            c, res = handle.dispatch_cgemm(ad * 2.0 ** -20, bd, SelectionPolicy(size_auto=1, size_tf32=1))
            assert "FP16TCEC_SCALED" in res.line, res.line
            e = relerr(c.cpu().numpy() * 2.0 ** 20, ref)
            assert e <= max(TOL_FACTOR * err_ref, 2e-7), (layout, "SCALED", e, err_ref)
    finally:
        handle.set_operand_layout("auto")
        handle.set_gemm_variant("auto")


@pytest.mark.parametrize("shape", [(512, 2048, 64), (512, 1024, 333), (1024, 4096, 1000)])
def test_operand_layout_a_multicast_bit_identical(handle, dev, shape):
    """In the A-expanded layout the multicast clusters still run the pair
    kernel's MMA sequence on the same operand bits: C is bit-identical."""
    m, n, k = shape
    a = matrix_recipe("uniform", m, k, 17 + m)
    b = matrix_recipe("uniform", k, n, 19 + n)
    ad, bd = torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev)
    outs = {}
    handle.set_operand_layout("a")
    try:
        for variant in ("wide", "wide_mc"):
            handle.set_gemm_variant(variant)
            c, _ = handle.cgemm(ad, bd, "TF32TCEC")
            outs[variant] = c.cpu().numpy()
    finally:
        handle.set_gemm_variant("auto")
        handle.set_operand_layout("auto")
    assert np.array_equal(outs["wide"].view(np.uint32), outs["wide_mc"].view(np.uint32))


def test_operand_layout_host_buffers(handle):
    """The host-buffer entry point with an A-expanded dispatch (m < n) equals
    the device-pointer dispatch bit for bit."""
    r = O.Rng(99)
    a, b = r.uniform_c32(384, 700), r.uniform_c32(700, 2100)
    cfg = make_config(SelectionPolicy(size_auto=64, size_tf32=32))
    ch, res_h = handle.dispatch_cgemm_host(a, b, cfg)
    dev = torch.device("cuda:0")
    cd, res_d = handle.dispatch_cgemm(torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev), cfg)
    assert res_h.line == res_d.line
    assert np.array_equal(ch.view(np.uint32), cd.cpu().numpy().view(np.uint32))


@pytest.mark.parametrize("shape", [(64, 1000, 33), (300, 257, 200), (512, 2048, 512), (130, 600, 1100)])
@pytest.mark.parametrize("mode", ["FP16TCEC", "TF32TCEC"])
def test_operand_layouts_bit_identical(handle, dev, shape, mode):
    """The two layouts hold the same products at the same K positions: A'(i, 2p)
    = Ar, A'(i, 2p+1) = Ai against B'(2q, ·) = (Br, -Bi), versus A''(2i, ·) = (Ar,
    -Ai) against B''(q, ·) = (Br, Bi) -- Ai*(-Bi) and (-Ai)*Bi are the same exact
    product (the splits are sign-symmetric) -- so the tensor core sums identical
    terms in identical order: C is bit-identical."""
    m, n, k = shape
    a = matrix_recipe("uniform", m, k, 31 + m)
    b = matrix_recipe("uniform", k, n, 37 + n)
    ad, bd = torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev)
    outs = {}
    try:
        for layout in ("a", "b"):
            handle.set_operand_layout(layout)
            c, _ = handle.cgemm(ad, bd, mode)
            outs[layout] = c.cpu().numpy()
    finally:
        handle.set_operand_layout("auto")
    assert np.array_equal(outs["a"].view(np.uint32), outs["b"].view(np.uint32))


@pytest.mark.parametrize("shape", [(512, 256, 64), (1024, 1000, 333), (2048, 512, 100), (768, 2048, 64),
                                   (4096, 2048, 512), (300, 5000, 40)])
@pytest.mark.parametrize("mode", ["FP16TCEC", "TF32TCEC", "AUTO", "SCALED"])
def test_pair_persistent_bit_identical_to_wide(handle, dev, shape, mode):
    """The persistent 256x128 pairs (two tiles' accumulators in TMEM) run the
    same MMA sequence per output as the 256x256 kernels -- the same k-blocks,
    the same RN flush per k-block, the same correction sum -- so C is
    bit-identical (no split-K on these shapes), ragged edges, the
    device-decided format and the descaled kind included."""
    m, n, k = shape
    a = matrix_recipe("uniform", m, k, 11 + m)
    b = matrix_recipe("uniform", k, n, 13 + n)
    if mode == "SCALED":
        a = (a * np.float32(2.0 ** -20)).astype(np.complex64)
    ad, bd = torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev)
    if mode in ("AUTO", "SCALED"):
        cfg = make_config(SelectionPolicy(size_auto=32, size_tf32=16))
    else:
        cfg = make_config(force=mode)
    outs, lines = {}, {}
    for variant in ("wide_persistent", "pair_persistent"):
        handle.set_gemm_variant(variant)
        try:
            c, res = handle.dispatch_cgemm(ad, bd, cfg)
            outs[variant] = c.cpu().numpy()
            lines[variant] = res.line
        finally:
            handle.set_gemm_variant("auto")
    assert lines["wide_persistent"] == lines["pair_persistent"]
    assert np.array_equal(outs["wide_persistent"].view(np.uint32), outs["pair_persistent"].view(np.uint32))


def test_randomized_shapes_variants_layouts_within_bar(handle, orc, dev):
    """Random ragged shapes (tile edges, k not a multiple of any k-block) on
    every tcgen05 variant and both operand layouts, FP16TCEC and TF32TCEC:
    relative error vs the f64 cgemm_oracle within the reference's bar
    (<= 4x the FP32_REF error, test_cgemm.cpp:64-66; 2e-6 floor for tiny k
    where FP32_REF is exact)."""
    rng = np.random.default_rng(989)
    variants = ["auto", "pair", "single", "wide", "wide_persistent", "pair_persistent"]
    try:
        for i in range(10):
            m, n = (int(x) for x in rng.integers(1, 700, 2))
            k = int(rng.integers(1, 600))
            a = matrix_recipe("uniform", m, k, 500 + i)
            b = matrix_recipe("uniform", k, n, 600 + i)
            ref = orc.cgemm_oracle(a, b)
            den = np.linalg.norm(ref)
            ad, bd = torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev)
            c32, _ = handle.cgemm(ad, bd, "FP32_REF")
            bar = max(4 * np.linalg.norm(c32.cpu().numpy().astype(np.complex128) - ref) / den, 2e-6)
            for mode in ("FP16TCEC", "TF32TCEC"):
                for layout in ("b", "a"):
                    handle.set_operand_layout(layout)
                    v = variants[i % len(variants)]
                    handle.set_gemm_variant(v)
                    c, _ = handle.cgemm(ad, bd, mode)
                    err = np.linalg.norm(c.cpu().numpy().astype(np.complex128) - ref) / den
                    assert err <= bar, ((m, n, k), mode, layout, v, err, bar)
    finally:
        handle.set_gemm_variant("auto")
        handle.set_operand_layout("auto")
