"""The headline configuration on the reference's own inputs (configs[1],
experiments.cpp:76-103): operands from Rng(1 + n) (A then B, uniform_pm1f),
default SelectionPolicy.  The device decision line must equal the reference
restatement's DecisionRecord line byte for byte (precsel.cpp:275-297,
185-205), and the AUTO result must meet the reference's accuracy bar -- rel.
error <= 4x the FP32_REF error and <= 5e-6 (test_cgemm.cpp:64-66,
SPEC.md:588) -- on sampled rows against the f64 cgemm_oracle."""
import numpy as np
import pytest
import torch

import oracle as O
from paper_2303_08989_b200 import make_config
from paper_2303_08989_b200.workload import sweep_operands

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n", [2048, 4096, 8192, 16384])
def test_reference_inputs_decision_line(handle, orc, dev, n):
    a_h, b_h = sweep_operands(n)
    a, b = a_h.to(dev), b_h.to(dev)
    _, res = handle.dispatch_cgemm(a, b, make_config())
    rc, want = orc.dispatch_decision(a_h.numpy(), b_h.numpy(), O.make_config())
    assert rc == 0
    assert res.line == want.line.decode(), (res.line, want.line)
    assert (res.kind, res.scale_a, res.scale_b) == (want.kind, want.scale_a, want.scale_b)
    for s_dev, s_ref in ((res.stats_a, want.stats_a), (res.stats_b, want.stats_b)):
        assert (s_dev.n1, s_dev.n2, s_dev.n_nonzero, s_dev.n_total) == \
               (s_ref.n1, s_ref.n2, s_ref.n_nonzero, s_ref.n_total)


@pytest.mark.parametrize("n", [4096, 8192])
def test_reference_inputs_accuracy_bar(handle, orc, dev, n):
    a_h, b_h = sweep_operands(n)
    a, b = a_h.to(dev), b_h.to(dev)
    c, res = handle.dispatch_cgemm(a, b, make_config())
    rows = np.sort(np.random.default_rng(n).choice(n, 24, replace=False))
    ref = orc.cgemm_oracle(a_h.numpy()[rows], b_h.numpy())
    got = c[torch.from_numpy(rows).to(dev)].cpu().numpy().astype(np.complex128)
    c32, _ = handle.cgemm(a[torch.from_numpy(rows).to(dev)].contiguous(), b, "FP32_REF")
    den = np.linalg.norm(ref)
    err = np.linalg.norm(got - ref) / den
    err32 = np.linalg.norm(c32.cpu().numpy().astype(np.complex128) - ref) / den
    assert err <= 4 * err32, (res.line, err, err32)
    assert err <= 5e-6, (res.line, err)
