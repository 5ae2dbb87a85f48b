"""The reference's OWN C++ test programs, compiled unchanged against the B200
drop-in (include/mpsgemm/*.hpp -> include/mpsgemm_b200.hpp, linked to
libtcec_b200.so; oracle/Makefile target `reftests`, built where
/root/reference exists and shipped with the repo snapshot):

  test_cgemm.cpp    cgemm / cgemm_batched / cgemm_oracle / relative_error
  test_precsel.cpp  exp_stats[_staged], matrix_tolerance, select_mode, scaling,
                    dispatch_cgemm routing, decision log, concurrency
  test_tensor.cpp   permute, contract_pair / contract_network, greedy_path,
                    validate_network, random_network, save/load_network
  test_qcircuit.cpp circuits, circuit_to_network, amplitude, state-vector oracle

On the GPU box every program must report zero failed test cases."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "reftests")
PROGRAMS = ["test_cgemm", "test_precsel", "test_tensor", "test_qcircuit"]


def _exe(name):
    p = os.path.join(BIN, name)
    if not os.path.exists(p):
        pytest.skip("reference test programs not built here (oracle/Makefile reftests needs /root/reference)")
    return p


@pytest.mark.parametrize("name", PROGRAMS)
def test_reference_program_links_to_the_drop_in(name):
    r = subprocess.run(["ldd", _exe(name)], capture_output=True, text=True)
    assert "libtcec_b200.so" in r.stdout and "not found" not in r.stdout, r.stdout


@pytest.mark.gpu
@pytest.mark.parametrize("name", PROGRAMS)
def test_reference_program_passes_on_b200(name):
    r = subprocess.run([_exe(name)], capture_output=True, text=True, timeout=900)
    out = r.stdout + r.stderr
    assert r.returncode == 0 and "| 0 failed |" in out, out[-4000:]
