"""Relative errors of the Sycamore-layout amplitudes vs contract_network_oracle
(the quantities tests/test_gpu_sycamore.py bounds)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_2303_08989_b200 import Handle, make_config  # noqa: E402
from paper_2303_08989_b200.circuits import circuit_to_network, sycamore_like  # noqa: E402
from paper_2303_08989_b200.network import Network  # noqa: E402
from paper_2303_08989_b200.slicing import (SlicePlan, assignment, device_evaluator, find_slices,  # noqa: E402
                                           slice_spec, sliced_amplitude)

h = Handle(0)
for cyc in (10, 12):
    circ = sycamore_like(cyc, 1)
    spec = circuit_to_network(circ, [(q * 7 + 3) % 2 for q in range(circ.n_qubits)])
    path, sliced, _ = bench.load_or_build_plan(spec, cyc, "plan")
    if cyc == 10:
        sliced = find_slices(spec, path, n_labels=2)
    plan = SlicePlan.build(spec, path, sliced)
    net = Network(h, plan.base)
    for label, cfg in (("AUTO-0", make_config()), ("FP32_BASELINE", make_config(force="FP32_REF"))):
        amp, full = sliced_amplitude(device_evaluator(net, plan, cfg), plan)
        errs = []
        for s in (0, plan.n_slices - 1):
            onet = Network(h, slice_spec(spec, plan.sliced, assignment(s, plan.dims)))
            z = complex(onet.contract_oracle(path).data.reshape(-1)[0])
            onet.close()
            errs.append(abs(complex(full[s]) - z) / abs(z))
        print(f"m={cyc} {plan.n_slices} slices {label}: slice rel err {errs[0]:.2e} / {errs[1]:.2e}", flush=True)
    net.close()
