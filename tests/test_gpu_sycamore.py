"""The north-star path end to end at a size a test can afford: a 53-qubit
Sycamore-layout circuit (sycamore_like(10, 1), bench.py --workload sycamore
--cycles 10) along the committed contraction plan, sliced over 4 slices and
evaluated through the slice scheduler on the device (AUTO-0: tensor-core
steps with device-side selection, fused TTGT gathers, skinny FP32-tier
kernels), against contract_network_oracle of the unsliced network along the
same path (network.cpp:179-186; the f64 fold on the device, pinned
bit-identical to the reference's CPU oracle by
test_device_f64_oracle_is_the_reference_oracle)."""
import os
import sys

import numpy as np
import pytest

from paper_2303_08989_b200 import make_config
from paper_2303_08989_b200.circuits import circuit_to_network, sycamore_like
from paper_2303_08989_b200.network import Network
from paper_2303_08989_b200.slicing import SlicePlan, device_evaluator, find_slices, sliced_amplitude

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def syc10():
    sys.path.insert(0, ROOT)
    import bench
    circ = sycamore_like(10, 1)
    spec = circuit_to_network(circ, [(q * 7 + 3) % 2 for q in range(circ.n_qubits)])
    path, _, kind = bench.load_or_build_plan(spec, 10, "plan")
    assert kind.startswith("hyper (cached"), kind
    return spec, path


def test_sycamore_m10_sliced_amplitude_vs_f64_oracle(handle, syc10):
    spec, path = syc10
    onet = Network(handle, spec)
    z = complex(onet.contract_oracle(path).data.reshape(-1)[0])
    onet.close()
    assert abs(z) > 0
    plan = SlicePlan.build(spec, path, find_slices(spec, path, n_labels=2))
    assert plan.n_slices == 4
    net = Network(handle, plan.base)
    errs = {}
    for label, cfg in (("AUTO-0", make_config()), ("FP32_BASELINE", make_config(force="FP32_REF"))):
        amp, full = sliced_amplitude(device_evaluator(net, plan, cfg), plan)
        assert len(full) == 4 and np.all(np.isfinite(np.asarray(full)))
        errs[label] = abs(complex(amp) - z) / abs(z)
    net.close()
    # the paper's claim: AUTO keeps FP32-level accuracy (measured 3-4e-6 here)
    assert errs["FP32_BASELINE"] <= 3e-5, errs
    assert errs["AUTO-0"] <= 3e-5, errs


def test_sycamore_m12_slices_vs_f64_oracle(handle):
    """configs[3] itself (m = 12, the committed 32-slice plan): every slice value
    through the device slice scheduler (AUTO-0), slice 0 and slice 31 against
    contract_network_oracle of that slice along the same path."""
    sys.path.insert(0, ROOT)
    import bench
    from paper_2303_08989_b200.slicing import assignment, slice_spec
    circ = sycamore_like(12, 1)
    spec = circuit_to_network(circ, [(q * 7 + 3) % 2 for q in range(circ.n_qubits)])
    path, sliced, kind = bench.load_or_build_plan(spec, 12, "plan")
    assert kind.startswith("hyper (cached"), kind
    plan = SlicePlan.build(spec, path, sliced)
    assert plan.n_slices == 32
    net = Network(handle, plan.base)
    amp, full = sliced_amplitude(device_evaluator(net, plan, make_config()), plan)
    net.close()
    full = np.asarray(full)
    assert full.shape == (32,) and np.all(np.isfinite(full))
    for s in (0, 31):
        onet = Network(handle, slice_spec(spec, plan.sliced, assignment(s, plan.dims)))
        z = complex(onet.contract_oracle(path).data.reshape(-1)[0])
        onet.close()
        assert abs(complex(full[s]) - z) <= 3e-5 * abs(z), (s, full[s], z)
    assert abs(complex(amp) - complex(np.sum(full.astype(np.complex128)))) <= 1e-12 * max(1.0, abs(amp))
