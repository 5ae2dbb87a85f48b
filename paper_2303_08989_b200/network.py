"""Tensor-network contraction through the C-ABI (host mirror of network.hpp).

    net = Network(handle, spec)                  # TensorNetwork (network.hpp:17-19)
    path = net.greedy_path()                     # greedy_path (network.hpp:49)
    t = net.contract(path, config)               # contract_network (network.hpp:37-38)
    z = amplitude(handle, circuit, x, config)    # amplitude (qcircuit.hpp:49-52)

String labels are mapped to integer ids at the boundary; the label order and
the SSA node numbering of paths are the reference's.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import ExtentMismatch, ShapeMismatch, check
from .api import Handle, SelectionPolicy, make_config
from .circuits import Circuit, NetworkSpec, circuit_to_network


@dataclass
class Tensor:
    """Tensor<std::complex<float>> (tensor.hpp:16-53)."""
    labels: list
    dims: list
    data: np.ndarray  # complex64, row-major in label order


def _cfg(config):
    if config is None or isinstance(config, SelectionPolicy):
        return make_config(config)
    return config


class Network:
    def __init__(self, handle: Handle | None, spec: NetworkSpec):
        """handle=None builds a planning-only network (greedy_path works without a GPU)."""
        self.handle = handle
        self.lib = handle.lib if handle is not None else _lib.load()
        self.spec = spec
        self.label_ids: dict[str, int] = {}
        ranks, labels, dims = [], [], []
        for ls, ds in zip(spec.labels, spec.dims):
            ranks.append(len(ls))
            for l, d in zip(ls, ds):
                labels.append(self.label_ids.setdefault(l, len(self.label_ids)))
                dims.append(int(d))
        self.names = {v: k for k, v in self.label_ids.items()}
        n = len(ranks)
        r = (C.c_int * max(n, 1))(*ranks)
        lab = (C.c_int * max(len(labels), 1))(*labels)
        dm = (C.c_int64 * max(len(dims), 1))(*dims)
        net = C.c_void_p()
        check(self.lib.tcec_network_create(handle.h if handle is not None else None, n, r, lab,
                                           dm, C.byref(net)))
        self.net = net
        if handle is not None:
            handle._networks.add(self)
        self._steps_cache = None
        for i, d in enumerate(spec.data):
            self.set_node(i, d)

    def _steps(self, path):
        """ctypes view of a path's SSA pairs, cached for repeated calls with the
        same path object (batch loops call with one path many times)."""
        c = self._steps_cache
        if c is not None and c[0] is path and c[1] == len(path):
            return c[2], c[3]
        arr = np.ascontiguousarray(np.asarray(path, dtype=np.int32).reshape(-1))
        if arr.size == 0:
            arr = np.zeros(1, np.int32)
        ptr = arr.ctypes.data_as(C.POINTER(C.c_int))
        self._steps_cache = (path, len(path), arr, ptr)
        return arr, ptr

    def close(self):
        if getattr(self, "net", None):
            self.lib.tcec_network_destroy(self.net)
            self.net = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def n_nodes(self) -> int:
        return len(self.spec.labels)

    def set_node(self, i: int, data) -> None:
        d = np.ascontiguousarray(data, dtype=np.complex64)
        expect = int(np.prod(self.spec.dims[i])) if self.spec.dims[i] else 1
        if d.size != expect:
            raise _lib.ShapeMismatch(1, "tensor data length does not match dims")
        check(self.lib.tcec_network_set_node(self.net, i, d.ctypes.data_as(C.c_void_p)))

    def greedy_path(self):
        n = self.n_nodes
        buf = (C.c_int * max(2 * (n - 1), 1))()
        check(self.lib.tcec_network_greedy_path(self.net, buf))
        return [(buf[2 * i], buf[2 * i + 1]) for i in range(n - 1)]

    def contract(self, path, config=None, want_log: bool = False):
        """contract_network: returns Tensor (and the decision-log lines)."""
        cfg = _cfg(config)
        flat = [x for st in path for x in st]
        steps = (C.c_int * max(len(flat), 1))(*flat)
        cap = 1
        # output size bound: product of all open-label dims
        open_dims = {}
        for ls, ds in zip(self.spec.labels, self.spec.dims):
            for l, d in zip(ls, ds):
                open_dims[l] = d if l not in open_dims else None
        for d in open_dims.values():
            if d is not None:
                cap *= d
        out = np.empty(max(cap, 1), dtype=np.complex64)
        rank = C.c_int(0)
        labels = (C.c_int * max(len(open_dims), 1))()
        log = C.create_string_buffer(200 * (len(path) + 1)) if want_log else None
        check(self.lib.tcec_contract_network(self.net, steps, len(path), C.byref(cfg),
                                             out.ctypes.data_as(C.c_void_p), out.size,
                                             C.byref(rank), labels, log,
                                             len(log) if log is not None else 0))
        names = [self.names[labels[i]] for i in range(rank.value)]
        dims = []
        for nm in names:
            dims.append(next(d for ls, ds in zip(self.spec.labels, self.spec.dims)
                             for l, d in zip(ls, ds) if l == nm))
        size = int(np.prod(dims)) if dims else 1
        t = Tensor(names, dims, out[:size].copy())
        if want_log:
            lines = [ln for ln in log.value.decode().split("\n") if ln]
            return t, lines
        return t

    def contract_oracle(self, path) -> Tensor:
        """contract_network_oracle (network.hpp:39, network.cpp:179-186): the
        same TTGT fold with every value widened to complex128 and the
        reference's f64 GEMM order, computed on the device
        (tcec_contract_network_oracle; bit-identical to the reference's CPU
        oracle).  Returns a complex128 Tensor."""
        flat = [x for st in path for x in st]
        steps = (C.c_int * max(len(flat), 1))(*flat)
        open_dims = {}
        for ls, ds in zip(self.spec.labels, self.spec.dims):
            for l, d in zip(ls, ds):
                open_dims[l] = d if l not in open_dims else None
        cap = 1
        for d in open_dims.values():
            if d is not None:
                cap *= d
        out = np.empty(max(cap, 1), dtype=np.complex128)
        rank = C.c_int(0)
        labels = (C.c_int * max(len(open_dims), 1))()
        check(self.lib.tcec_contract_network_oracle(self.net, steps, len(path),
                                                    out.ctypes.data_as(C.c_void_p), out.size,
                                                    C.byref(rank), labels))
        names = [self.names[labels[i]] for i in range(rank.value)]
        dims = [next(d for ls, ds in zip(self.spec.labels, self.spec.dims) for l, d in zip(ls, ds)
                     if l == nm) for nm in names]
        size = int(np.prod(dims)) if dims else 1
        return Tensor(names, dims, out[:size].copy())

    def selector_batch(self, path, bitstrings, config=None, out=None) -> np.ndarray:
        """Amplitudes of many bitstrings over one plan / one captured graph.
        `bitstrings` / `out` may live in pinned host memory (faster copies)."""
        cfg = _cfg(config)
        _, steps = self._steps(path)
        sel = self.spec.selector_nodes
        nsel = len(sel)
        sel_arr = (C.c_int * max(nsel, 1))(*sel)
        bits = np.ascontiguousarray(np.asarray(bitstrings, dtype=np.uint8).reshape(-1))
        n = len(bitstrings)
        if out is None:
            out = np.empty(n, dtype=np.complex64)
        elif out.dtype != np.complex64 or out.size != n or not out.flags.c_contiguous:
            raise ValueError("out must be a contiguous complex64 array with one slot per bitstring")
        check(self.lib.tcec_contract_selector_batch(
            self.net, steps, len(path), C.byref(cfg), nsel, sel_arr, n,
            bits.ctypes.data_as(C.POINTER(C.c_uint8)), out.ctypes.data_as(C.c_void_p)))
        return out


    def node_batch(self, path, var_nodes, runs, config=None) -> np.ndarray:
        """Closed-network values of many runs that differ only in the data of
        `var_nodes`; runs[r][i] is the data of var_nodes[i] in run r."""
        cfg = _cfg(config)
        _, steps = self._steps(path)
        nv = len(var_nodes)
        vn = (C.c_int * max(nv, 1))(*var_nodes)
        blocks = [np.ascontiguousarray(np.asarray(d, dtype=np.complex64).reshape(-1))
                  for run in runs for d in run]
        data = np.concatenate(blocks) if blocks else np.zeros(1, np.complex64)
        out = np.empty(max(len(runs), 1), dtype=np.complex64)
        check(self.lib.tcec_contract_node_batch(self.net, steps, len(path), C.byref(cfg), nv, vn,
                                                len(runs), data.ctypes.data_as(C.c_void_p),
                                                out.ctypes.data_as(C.c_void_p)))
        return out[:len(runs)]

    def batch_run_info(self, run: int, n_steps: int | None = None):
        """(overflow flag, decision-log lines) of run `run` of the last batch
        (tcec_network_batch_run_info)."""
        steps = n_steps if n_steps is not None else max(self.n_nodes - 1, 1)
        ovf = C.c_int(0)
        log = C.create_string_buffer(200 * (steps + 1))
        check(self.lib.tcec_network_batch_run_info(self.net, int(run), C.byref(ovf), log, len(log)))
        return bool(ovf.value), [ln for ln in log.value.decode().split("\n") if ln]


def _fmt9(v: float) -> str:
    """printf("%.9g") of a float widened to double (network.cpp:451-453)."""
    return "%.9g" % float(v)


def save_network(spec: NetworkSpec) -> str:
    """save_network text format (network.hpp:62-66, network.cpp:440-458): per node
    "node <id> labels l1,l2 dims d1,d2" ("-" for rank 0), then the values as
    "%.9g %.9g" pairs (an exact round trip for f32)."""
    out = []
    for i, (ls, ds, d) in enumerate(zip(spec.labels, spec.dims, spec.data)):
        lab = ",".join(str(x) for x in ls) if ls else "-"
        dim = ",".join(str(int(x)) for x in ds) if ds else "-"
        out.append(f"node {i} labels {lab} dims {dim}\n")
        v = np.asarray(d, dtype=np.complex64).reshape(-1)
        out.append(" ".join(f"{_fmt9(z.real)} {_fmt9(z.imag)}" for z in v) + "\n")
    return "".join(out)


def load_network(text: str) -> NetworkSpec:
    """load_network (network.cpp:472-501): the inverse of save_network,
    validated like validate_network."""
    tok = text.split()
    spec = NetworkSpec()
    i = 0
    while i < len(tok):
        if tok[i] != "node":
            raise ShapeMismatch(1, "expected 'node' header, got: " + tok[i])
        if i + 5 >= len(tok) or tok[i + 2] != "labels" or tok[i + 4] != "dims":
            raise ShapeMismatch(1, "malformed node header")
        labels = [] if tok[i + 3] == "-" else tok[i + 3].split(",")
        dims = [] if tok[i + 5] == "-" else [int(x) for x in tok[i + 5].split(",")]
        i += 6
        n = int(np.prod(dims)) if dims else 1
        if i + 2 * n > len(tok):
            raise ShapeMismatch(1, "truncated tensor data")
        vals = np.array([float(x) for x in tok[i:i + 2 * n]], dtype=np.float64).astype(np.float32)
        i += 2 * n
        spec.labels.append(labels)
        spec.dims.append(dims)
        spec.data.append(vals.view(np.complex64).reshape(dims if dims else [1]))
    occ = {}
    for ls, ds in zip(spec.labels, spec.dims):
        for l, d in zip(ls, ds):
            occ.setdefault(l, []).append(d)
    for l, ds in occ.items():
        if len(ds) > 2:
            raise ShapeMismatch(1, f"label {l} appears in more than two nodes")
        if len(ds) == 2 and ds[0] != ds[1]:
            raise ExtentMismatch(5, f"label {l} has mismatched extents")
    return spec


def contract_pair(handle: Handle, a: Tensor, b: Tensor, config=None) -> Tensor:
    """contract_pair (network.hpp:29-32) as a two-node fold."""
    spec = NetworkSpec(labels=[list(a.labels), list(b.labels)], dims=[list(a.dims), list(b.dims)],
                       data=[a.data, b.data])
    net = Network(handle, spec)
    try:
        return net.contract([(0, 1)], config)
    finally:
        net.close()


def statevector_oracle(handle: Handle, circuit: Circuit):
    """statevector_oracle (qcircuit.hpp:56, qcircuit.cpp:197-225): the f64 state
    vector of |0...0> under the circuit, on the device (tcec_statevector_f64,
    the reference's gate order and complex arithmetic -> bit-identical); qubit q
    is bit q of the index.  Returns a complex128 CUDA tensor."""
    import torch
    from .circuits import CZ, gate_matrix, validate_circuit
    validate_circuit(circuit)
    if circuit.n_qubits > 24:
        raise _lib.TooManyQubits(11, "state-vector oracle limited to 24 qubits")
    qa, qb, u = [], [], []
    for layer in circuit.layers:
        for g in layer:
            if g.kind == CZ:
                qa.append(g.qubits[0])
                qb.append(g.qubits[1])
                u.extend([0.0] * 8)
                continue
            if len(g.qubits) != 1:
                raise ValueError(f"statevector_oracle: gate {g.kind} is not in the reference gate set")
            m = gate_matrix(g.kind)
            qa.append(g.qubits[0])
            qb.append(-1)
            u.extend(v for z in m for v in (z.real, z.imag))
    n = len(qa)
    st = torch.empty(1 << circuit.n_qubits, dtype=torch.complex128, device=torch.device("cuda", handle.device))
    ia = (C.c_int * max(n, 1))(*qa)
    ib = (C.c_int * max(n, 1))(*qb)
    du = (C.c_double * max(8 * n, 8))(*u)
    handle._ordered_call(handle.lib.tcec_statevector_f64, handle.h, circuit.n_qubits, n, ia, ib, du,
                         C.c_void_p(st.data_ptr()))
    return st


def amplitude(handle: Handle, circuit: Circuit, x, config=None) -> np.complex64:
    """amplitude (qcircuit.cpp:184-195): network -> greedy path -> contraction."""
    net = Network(handle, circuit_to_network(circuit, x))
    try:
        return net.contract(net.greedy_path(), config).data[0]
    finally:
        net.close()
