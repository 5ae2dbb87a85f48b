"""Device-side precision selection + dispatch (reference test_precsel.cpp:242-349).

The exponent statistics, tolerance levels, chosen mode, scale exponents and the
decision-log line must be identical to the reference (golden + oracle); the
FP32 tier output is bit-identical, the tensor-core tiers are within tolerance."""
import numpy as np
import pytest
import torch

import oracle as O
from paper_2303_08989_b200 import SelectionPolicy, make_config
from tests.conftest import bits
from tests.golden.recipes import matrix_recipe

pytestmark = pytest.mark.gpu


def relerr(c, ref):
    return float(np.linalg.norm(np.asarray(c, np.complex128) - ref) / np.linalg.norm(ref))


def _gpu_cfg(kw):
    kw = dict(kw)
    force = kw.pop("force", None)
    pol = SelectionPolicy(**{k: v for k, v in kw.items()})
    return make_config(pol, force=force)


def test_dispatch_golden(handle, orc, golden, dev):
    for d in golden("dispatch.json"):
        a = matrix_recipe(d["a"], d["m"], d["k"], d["seed_a"])
        b = matrix_recipe(d["b"], d["k"], d["n"], d["seed_b"])
        c, res = handle.dispatch_cgemm(torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev),
                                       _gpu_cfg(d["cfg"]))
        assert res.line == d["line"], (d["cfg"], res.line, d["line"])
        assert (["FP16TCEC", "FP16TCEC_SCALED", "TF32TCEC", "FP32_BASELINE"][res.kind],
                res.scale_a, res.scale_b) == (d["kind"], d["scale_a"], d["scale_b"])
        assert bool(res.overflow) == bool(d["overflow"])
        ch = c.cpu().numpy()
        rc, co, _ = orc.dispatch_cgemm(a, b, O.make_config(**d["cfg"]))
        if d["kind"] == "FP32_BASELINE" or d["cfg"].get("force") in ("FP32_REF", "FP64_ORACLE"):
            assert np.array_equal(bits(ch.view(np.float32)), bits(co.view(np.float32)))
        elif d["c_oracle"] is not None and "TC" not in str(d["cfg"].get("force", "")).replace("TCEC", ""):
            ref = np.array(d["c_oracle"], np.float64).view(np.complex128).reshape(d["m"], d["n"])
            assert relerr(ch, ref) <= max(4 * relerr(co, ref), 5e-7)


def test_default_policy_routing(handle, dev):
    # SPEC.md:596 acceptance 10 (shapes scaled to keep the test fast) + test_precsel.cpp:242-256
    small = torch.from_numpy(matrix_recipe("uniform", 64, 64, 410)).to(dev)
    _, r = handle.dispatch_cgemm(small, small)
    assert r.line == "64,64,64,FP32_BASELINE,0,0,-,-,-,-,-,-" and not r.has_stats
    mid = torch.from_numpy(matrix_recipe("uniform", 512, 512, 411)).to(dev)
    _, r = handle.dispatch_cgemm(mid, mid)
    assert r.line.startswith("512,512,512,TF32TCEC,0,0,-,-,-,-,-,-")
    big = torch.from_numpy(matrix_recipe("uniform", 2048, 2048, 412)).to(dev)
    _, r = handle.dispatch_cgemm(big, big)
    assert r.has_stats and r.line.split(",")[3] in ("FP16TCEC_SCALED", "FP16TCEC")


@pytest.mark.parametrize("recipe,t,want", [
    ("banded", 0.0, "FP16TCEC"),
    ("tiny20", 0.0, "FP16TCEC_SCALED"),
    ("uniform", 0.0, "FP16TCEC_SCALED"),
    ("uniform", 0.1, "FP16TCEC"),
    ("type3", 0.0, "TF32TCEC"),
    ("type3", 0.5, "FP16TCEC_SCALED"),
])
def test_auto_selection_outcomes(handle, orc, dev, recipe, t, want):
    a = matrix_recipe(recipe, 96, 88, 71)
    b = matrix_recipe("banded" if recipe == "type3" else recipe, 88, 80, 72)
    cfg_kw = dict(threshold_t=t, size_auto=16, size_tf32=8)
    c, res = handle.dispatch_cgemm(torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev),
                                   _gpu_cfg(cfg_kw))
    rc, co, ro = orc.dispatch_cgemm(a, b, O.make_config(**cfg_kw))
    assert res.line == ro.line.decode()
    assert res.line.split(",")[3] == want
    ref = orc.cgemm_oracle(a, b)
    err_ref = relerr(orc.cgemm(a, b, "FP32_REF")[0], ref)
    assert relerr(c.cpu().numpy(), ref) <= max(4 * err_ref, 5e-7)


def test_scaled_fp16_stays_accurate_on_tiny_inputs(handle, orc, dev):
    # test_precsel.cpp:278-289: e_max = -20 -> scale 34, error <= 1e-6
    r = O.Rng(411)
    a = (r.uniform_c32(16, 16) * np.float32(0.5) + np.complex64(1 + 1j)) * np.float32(2.0 ** -20)
    b = (r.uniform_c32(16, 16) * np.float32(0.5) + np.complex64(1 + 1j)) * np.float32(2.0 ** -20)
    c, res = handle.dispatch_cgemm(torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev),
                                   SelectionPolicy(size_auto=16, size_tf32=8))
    assert res.line.split(",")[3] == "FP16TCEC_SCALED" and res.scale_a == 34
    assert relerr(c.cpu().numpy(), orc.cgemm_oracle(a, b)) <= 1e-6


def test_forced_fp16_underflows_on_type2_like_inputs(handle, orc, dev):
    """SPEC.md:593 criterion 5: forced FP16TCEC on 1e-8-scale inputs loses the
    result, the selector's scaled mode does not."""
    a = matrix_recipe("uniform", 64, 64, 5) * np.float32(1e-8)
    b = matrix_recipe("uniform", 64, 64, 6) * np.float32(1e-8)
    ad, bd = torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev)
    ref = orc.cgemm_oracle(a, b)
    forced, _ = handle.cgemm(ad, bd, "FP16TCEC")
    assert np.abs(forced.cpu().numpy()).max() < 1e-3 * np.abs(ref).max()
    c, res = handle.dispatch_cgemm(ad, bd, SelectionPolicy(size_auto=16, size_tf32=8))
    assert res.line.split(",")[3] == "FP16TCEC_SCALED"
    assert relerr(c.cpu().numpy(), ref) < 1e-6


def test_scaled_roundtrip_bit_exact(handle, dev):
    # test_precsel.cpp:226-240: descale(cgemm(scale A, scale B)) == cgemm(A, B) bit for bit
    g = np.random.default_rng(409)
    def band(r, c):
        v = (g.choice([-1.0, 1.0], (r, c, 2)) * (0.25 + 0.7 * g.random((r, c, 2)))).astype(np.float32)
        return np.ascontiguousarray(v.view(np.complex64)[..., 0])
    a, b = band(24, 16), band(16, 20)
    ad, bd = torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev)
    direct, _ = handle.cgemm(ad, bd, "FP16TCEC")
    scaled, _ = handle.cgemm(handle.scale_matrix(ad, 3), handle.scale_matrix(bd, 5), "FP16TCEC")
    handle.descale_output_inplace(scaled, 3, 5)
    assert torch.equal(scaled, direct)


def test_forced_modes(handle, orc, dev):
    a = matrix_recipe("uniform", 8, 8, 412)
    b = matrix_recipe("uniform", 8, 8, 413)
    ad, bd = torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev)
    for f in O.FORCED:
        c, res = handle.dispatch_cgemm(ad, bd, make_config(force=f))
        assert res.line.split(",")[3] == f
        if f == "FP16TCEC_SCALED":
            assert res.has_stats
            assert relerr(c.cpu().numpy(), orc.cgemm_oracle(a, b)) <= 1e-5


def test_host_buffer_entry_point(handle, orc):
    a = matrix_recipe("uniform", 200, 150, 1)
    b = matrix_recipe("uniform", 150, 120, 2)
    c, res = handle.dispatch_cgemm_host(a, b, make_config(force="FP32_REF"))
    co, _ = orc.cgemm(a, b, "FP32_REF")
    assert np.array_equal(bits(c.view(np.float32)), bits(co.view(np.float32)))
    c2, res2 = handle.dispatch_cgemm_host(a, b, SelectionPolicy(size_auto=64, size_tf32=32))
    rc, _, ro = orc.dispatch_cgemm(a, b, O.make_config(size_auto=64, size_tf32=32))
    assert res2.line == ro.line.decode()


def test_host_buffer_row_chunks_match_the_device_path(handle, dev):
    """The host-buffer entry point runs the wide GEMM in row chunks and copies
    finished rows back while the next chunk computes; every tile is the same
    computation, so C is bit-identical to the one-launch device dispatch."""
    g = np.random.default_rng(12)
    m, n, k = 8448, 1536, 640
    a = (g.random((m, k, 2), dtype=np.float32) * 2 - 1).view(np.complex64)[..., 0].copy()
    b = (g.random((k, n, 2), dtype=np.float32) * 2 - 1).view(np.complex64)[..., 0].copy()
    pol = SelectionPolicy(size_auto=512, size_tf32=256)
    c_host, res_h = handle.dispatch_cgemm_host(a, b, pol)
    c_dev, res_d = handle.dispatch_cgemm(torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev), pol)
    assert res_h.line == res_d.line
    assert np.array_equal(c_host.view(np.uint32), c_dev.cpu().numpy().view(np.uint32))


@pytest.mark.parametrize("shape", [(16384, 768, 384), (8448, 2304, 640)])
@pytest.mark.parametrize("case", ["uniform", "late_outlier", "late_tiny", "first_outlier", "late_b_outlier",
                                  "sample_predicts_tiny",
                                  "FP16TCEC", "TF32TCEC", "FP16TCEC_SCALED", "fp16_overflow"])
def test_host_pipeline_matches_the_device_path(handle, dev, case, shape):
    """Large host-buffer dispatches copy A in row chunks and start each chunk's
    GEMM under a decision taken from B and the first chunk; the exact decision
    follows, and a disagreement reruns the plain path.  Either way C and the
    decision record are bit-identical to the device-buffer dispatch -- including
    inputs whose later rows change the decision (late outlier / late tiny rows)."""
    g = np.random.default_rng(21)
    m, n, k = shape  # n = 2304: B in six column parts of 384, three sent after A; n = 768: three of 256
    a = (g.random((m, k, 2), dtype=np.float32) * 2 - 1).view(np.complex64)[..., 0].copy()
    b = (g.random((k, n, 2), dtype=np.float32) * 2 - 1).view(np.complex64)[..., 0].copy()
    pol = SelectionPolicy(size_auto=128, size_tf32=64)
    if case == "late_outlier":
        a[m - 5, 7] = 3.0e20 + 1.0e20j
    elif case == "late_tiny":
        a[m // 2:] *= np.float32(2.0 ** -30)
    elif case == "first_outlier":
        a[3, 2] = 1.0e6
    elif case == "late_b_outlier":
        b[k // 2, n - 3] = 2.0e9 - 1.0e9j
    elif case == "sample_predicts_tiny":
        # the first A chunk (the speculation's sample, 1024 rows) holds many
        # components just above the stage-2 threshold 2^-29 (2^-26 < 2^(-29 + 5))
        # but none below it; later rows hold some below it (exact: TF32).  The
        # density extrapolation must predict TF32 -> no rerun.
        sel = g.random((1024, k)) < 0.1
        a[:1024][sel] = np.complex64(2.0 ** -26 + 2.0 ** -26 * 1j)
        a[m - 7, 5] = np.complex64(2.0 ** -35)
    elif case == "fp16_overflow":
        a[m - 100, 3] = 9.0e4
        pol = make_config(force="FP16TCEC")
    elif case in ("FP16TCEC", "TF32TCEC", "FP16TCEC_SCALED"):
        pol = make_config(force=case)
    runs0, reruns0 = handle.host_pipeline_stats()
    c_host, res_h = handle.dispatch_cgemm_host(a, b, pol)
    runs1, reruns1 = handle.host_pipeline_stats()
    assert runs1 == runs0 + 1  # m >= 8192 on the tensor-core tier: pipelined
    if case in ("late_outlier", "late_b_outlier"):
        assert reruns1 == reruns0 + 1  # the first parts could not predict the scale
    if case == "sample_predicts_tiny":
        assert reruns1 == reruns0  # the density extrapolation predicted the exact decision
    c_dev, res_d = handle.dispatch_cgemm(torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev), pol)
    if case in ("uniform", "late_outlier", "late_tiny", "late_b_outlier"):
        assert res_d.has_stats  # the AUTO tier: decided from statistics on the device
    assert res_h.line == res_d.line
    assert res_h.overflow == res_d.overflow
    assert np.array_equal(c_host.view(np.uint32), c_dev.cpu().numpy().view(np.uint32))
    # the same buffers again (the staging buffers and decision slots are reused)
    c_host2, res_h2 = handle.dispatch_cgemm_host(a, b, pol)
    assert res_h2.line == res_d.line
    assert np.array_equal(c_host2.view(np.uint32), c_host.view(np.uint32))


def test_empty_and_zero_operands(handle, dev):
    z = torch.zeros(32, 32, dtype=torch.complex64, device=dev)
    c, res = handle.dispatch_cgemm(z, z, SelectionPolicy(size_auto=16, size_tf32=8))
    assert res.line == "32,32,32,FP16TCEC,0,0,0,-,0,-,-,-"
    assert torch.count_nonzero(c) == 0
    a = torch.zeros(5, 0, dtype=torch.complex64, device=dev)
    b = torch.zeros(0, 7, dtype=torch.complex64, device=dev)
    for mode in ("FP32_REF", "FP16TCEC", "TF32TCEC"):
        c, _ = handle.cgemm(a, b, mode)
        assert c.shape == (5, 7) and torch.count_nonzero(c) == 0


def test_handles_on_concurrent_host_threads(dev):
    """Reentrancy (SURVEY.md 8(b) threading: pure and reentrant): one handle per
    host thread, dispatches and permutes issued concurrently (ctypes releases
    the GIL) give the bits of the same calls made serially."""
    import threading
    from paper_2303_08989_b200 import Handle
    g = np.random.default_rng(33)
    jobs = []
    for m, n, k in [(1024, 768, 512), (300, 200, 9000), (4096, 16, 8), (2048, 2048, 64)]:
        a = torch.from_numpy((g.random((m, k, 2), dtype=np.float32) * 2 - 1).view(np.complex64)[..., 0].copy()).to(dev)
        b = torch.from_numpy((g.random((k, n, 2), dtype=np.float32) * 2 - 1).view(np.complex64)[..., 0].copy()).to(dev)
        jobs.append((a, b))
    t = torch.randn(*([2] * 20), dtype=torch.complex64, device=dev)
    axes = [[int(v) for v in g.permutation(20)] for _ in range(4)]
    pol = SelectionPolicy(size_auto=64, size_tf32=32)

    def work(h, out):
        for a, b in jobs:
            c, res = h.dispatch_cgemm(a, b, pol)
            out.append((c.cpu(), res.line))
        for ax in axes:
            out.append((h.permute(t, ax).cpu(), ""))
        torch.cuda.synchronize()

    handles = [Handle(0) for _ in range(3)]
    serial = []
    work(handles[0], serial)
    outs = [[] for _ in handles]
    threads = [threading.Thread(target=work, args=(h, o)) for h, o in zip(handles, outs)]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    for o in outs:
        assert len(o) == len(serial)
        for (x, lx), (y, ly) in zip(o, serial):
            assert lx == ly
            assert torch.equal(x.view(torch.float32), y.view(torch.float32))
    for h in handles:
        h.close()


def test_graph_replay_reads_new_data(handle, orc, dev):
    """Small device-pointer dispatches replay a captured graph when the same
    pointers, shape and configuration come again: in-place changes to the
    operands (including ones that change the device decision) must show up
    exactly as in a fresh dispatch."""
    from paper_2303_08989_b200 import Handle
    g = np.random.default_rng(5)
    m, n, k = 384, 320, 256
    a_np = (g.random((m, k, 2), dtype=np.float32) * 2 - 1).view(np.complex64)[..., 0].copy()
    b_np = (g.random((k, n, 2), dtype=np.float32) * 2 - 1).view(np.complex64)[..., 0].copy()
    a, b = torch.from_numpy(a_np).to(dev), torch.from_numpy(b_np).to(dev)
    c = torch.empty(m, n, dtype=torch.complex64, device=dev)
    pol = SelectionPolicy(size_auto=128, size_tf32=64)
    fresh = Handle(0)
    for step in range(4):
        if step == 2:
            a.mul_(2.0 ** -20)  # moves e_max: another FP16TCEC_SCALED shift
        elif step == 3:
            a.copy_(torch.from_numpy((g.random((m, k, 2), dtype=np.float32) * 2 - 1)
                                     .view(np.complex64)[..., 0].copy()).to(dev))
        _, res = handle.dispatch_cgemm(a, b, pol, out=c)
        want, res_w = fresh.dispatch_cgemm(a.clone(), b.clone(), pol)
        assert res.line == res_w.line
        assert torch.equal(c.view(torch.float32), want.view(torch.float32))
        c32, _ = handle.dispatch_cgemm(a, b, make_config(force="FP32_REF"), out=c)
        ref, _ = orc.cgemm(a.cpu().numpy(), b.cpu().numpy(), "FP32_REF")
        assert np.array_equal(c32.cpu().numpy().view(np.uint32), ref.view(np.uint32))
    fresh.close()


def test_host_pipeline_on_a_caller_stream(dev):
    """The pipelined host-buffer dispatch on a handle bound to the caller's
    stream (tcec_set_stream) gives the bits of the handle's own stream, call
    after call (the staging buffers and side streams are reused)."""
    from paper_2303_08989_b200 import Handle
    g = np.random.default_rng(8)
    m, n, k = 8448, 2304, 640
    a = (g.random((m, k, 2), dtype=np.float32) * 2 - 1).view(np.complex64)[..., 0].copy()
    b = (g.random((k, n, 2), dtype=np.float32) * 2 - 1).view(np.complex64)[..., 0].copy()
    pol = SelectionPolicy(size_auto=128, size_tf32=64)
    h0 = Handle(0)
    want, res_w = h0.dispatch_cgemm_host(a, b, pol)
    h1 = Handle(0)
    s = torch.cuda.Stream(device=dev)
    h1.set_stream(s)
    for _ in range(2):
        got, res = h1.dispatch_cgemm_host(a, b, pol)
        assert res.line == res_w.line
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
    assert h1.host_pipeline_stats()[0] == 2
    h1.set_stream(None)
    h0.close()
    h1.close()


@pytest.mark.parametrize("shape", [(8448, 1536, 640), (300, 200, 100)])
@pytest.mark.parametrize("pinned", ["", "a", "b", "c", "abc"])
def test_host_buffers_pinned_or_pageable(handle, dev, shape, pinned):
    """Pageable host buffers (the C++ drop-in's std::vector storage) go through
    the pinned staging ring; any mix of pinned and pageable A / B / C gives the
    bits of the device-buffer dispatch, pipelined (m >= 8192) or not."""
    m, n, k = shape
    g = np.random.default_rng(5)

    def host(shape_, fill, pin):
        if pin:
            t = torch.empty(shape_, dtype=torch.complex64, pin_memory=True).numpy()
        else:
            t = np.empty(shape_, dtype=np.complex64)
        if fill:
            t.view(np.float32)[...] = g.random(t.view(np.float32).shape, dtype=np.float32) * 2 - 1
        return t

    a = host((m, k), True, "a" in pinned)
    b = host((k, n), True, "b" in pinned)
    c = host((m, n), False, "c" in pinned)
    pol = SelectionPolicy(size_auto=96, size_tf32=64)
    c_host, res_h = handle.dispatch_cgemm_host(a, b, pol, out=c)
    c_dev, res_d = handle.dispatch_cgemm(torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev), pol)
    assert res_h.line == res_d.line
    assert np.array_equal(c_host.view(np.uint32), c_dev.cpu().numpy().view(np.uint32))


def test_dispatch_decision_randomized_vs_oracle(handle, orc, dev):
    """Randomised selection parity (precsel.cpp:225-322): random shapes, input
    families, thresholds, targets, size gates and forced modes -- the device
    DecisionRecord line, kind and shifts equal the oracle's for every draw."""
    rng = np.random.default_rng(2303)
    recipes = ["uniform", "tiny20", "huge20", "banded", "type3", "subnormal", "mixed40", "ones", "zeros"]
    forced = [None] * 6 + ["FP32_REF", "FP64_ORACLE", "TF32TC", "FP16TC", "TF32TCEC", "FP16TCEC",
                           "FP16TCEC_SCALED"]
    for i in range(40):
        m, n, k = (int(x) for x in rng.integers(1, 97, 3))
        ra, rb = rng.choice(recipes, 2)
        a = matrix_recipe(str(ra), m, k, 1000 + i)
        b = matrix_recipe(str(rb), k, n, 2000 + i)
        t = float(rng.choice([0.0, 1e-6, 0.05, 0.3, 1.0]))
        target = int(rng.choice([0, 7, 14, 15, 20]))
        gate = int(rng.choice([1, 8, 32, 64, 4096]))
        gate32 = int(rng.choice([1, gate]))
        force = forced[int(rng.integers(0, len(forced)))]
        kw = dict(threshold_t=t, size_auto=gate, size_tf32=min(gate32, gate), target=target, force=force)
        gkw = dict(threshold_t=t, size_auto=gate, size_tf32=min(gate32, gate), target_max_exponent=target,
                   force=force)
        try:
            _, res = handle.dispatch_cgemm(torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev),
                                           _gpu_cfg(gkw))
            got = (0, res.line, res.kind, res.scale_a, res.scale_b)
        except Exception as e:  # noqa: BLE001 -- the reference's exceptions map to error codes
            got = (type(e).__name__,)
        rc, want = orc.dispatch_decision(a, b, O.make_config(**kw))
        if rc == 0:
            assert got == (0, want.line.decode(), want.kind, want.scale_a, want.scale_b), (i, kw, ra, rb, got)
        else:
            assert got[0] != 0, (i, kw, ra, rb, rc, got)
