"""Random-circuit workload and its tensor network (host side).

Restates the reference's deterministic generators so the B200 path contracts
exactly the reference's networks:
  * Rng          -- rng.hpp:13-56 (std::mt19937_64 + hand-rolled distributions)
  * gate_matrix  -- qcircuit.cpp:48-61;  gate_tensor -- qcircuit.cpp:63-81
  * cz_pattern   -- qcircuit.cpp:83-102; rqc_rectangular -- qcircuit.cpp:104-140
  * circuit_to_network -- qcircuit.cpp:142-182 (wire labels "w<q>_<step>")
This is workload generation (host planning, out of the device hot path).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

_M64 = (1 << 64) - 1


class Mt19937_64:
    """std::mt19937_64 ([rand.predef]): w=64, n=312, m=156, r=31."""

    N, M = 312, 156
    A = 0xB5026F5AA96619E9
    UM, LM = 0xFFFFFFFF80000000, 0x7FFFFFFF

    def __init__(self, seed: int):
        mt = [0] * self.N
        mt[0] = seed & _M64
        for i in range(1, self.N):
            mt[i] = (6364136223846793005 * (mt[i - 1] ^ (mt[i - 1] >> 62)) + i) & _M64
        self.mt = mt
        self.idx = self.N

    def _twist(self):
        mt, N, M = self.mt, self.N, self.M
        for i in range(N):
            x = (mt[i] & self.UM) | (mt[(i + 1) % N] & self.LM)
            xa = x >> 1
            if x & 1:
                xa ^= self.A
            mt[i] = mt[(i + M) % N] ^ xa
        self.idx = 0

    def __call__(self) -> int:
        if self.idx >= self.N:
            self._twist()
        x = self.mt[self.idx]
        self.idx += 1
        x ^= (x >> 29) & 0x5555555555555555
        x ^= (x << 17) & 0x71D67FFFEDA60000
        x ^= (x << 37) & 0xFFF7EEE000000000
        x ^= x >> 43
        return x & _M64


class Rng:
    """rng.hpp:13-56."""

    def __init__(self, seed: int):
        self.eng = Mt19937_64(seed)
        self._spare = 0.0
        self._have_spare = False

    def next_u64(self) -> int:
        return self.eng()

    def next_below(self, n: int) -> int:
        limit = n * (_M64 // n)
        v = self.eng()
        while v >= limit:
            v = self.eng()
        return v % n

    def uniform01(self) -> float:
        return float(self.eng() >> 11) * 2.0 ** -53

    def uniform01_pos(self) -> float:
        return float((self.eng() >> 11) + 1) * 2.0 ** -53

    def uniform_pm1f(self) -> np.float32:
        return np.float32(2.0 * self.uniform01() - 1.0)

    def gaussian(self, stddev: float) -> float:
        if self._have_spare:
            self._have_spare = False
            return self._spare * stddev
        u1 = self.uniform01_pos()
        u2 = self.uniform01()
        r = math.sqrt(-2.0 * math.log(u1))
        a = 6.283185307179586476925286766559 * u2
        self._spare = r * math.sin(a)
        self._have_spare = True
        return r * math.cos(a) * stddev

    def uniform_c32(self, rows: int, cols: int) -> np.ndarray:
        """experiments.cpp:27-31 random_uniform_matrix (re then im per element)."""
        out = np.empty(rows * cols * 2, dtype=np.float32)
        for i in range(out.size):
            out[i] = self.uniform_pm1f()
        return out.view(np.complex64).reshape(rows, cols)


# ------------------------------------------------------------------ gates
H, T, SX, SY, CZ = "H", "T", "SX", "SY", "CZ"
SW, FSIM = "SW", "FSIM"  # Sycamore-class extension (not in the reference gate set)
_SINGLES = (T, SX, SY)
TWO_QUBIT = (CZ, FSIM)


def gate_matrix(kind: str) -> np.ndarray:
    """qcircuit.cpp:48-61 (f64, row-major)."""
    s = 1.0 / math.sqrt(2.0)
    if kind == H:
        return np.array([s, s, s, -s], dtype=np.complex128)
    if kind == T:
        return np.array([1.0, 0.0, 0.0, complex(s, s)], dtype=np.complex128)
    if kind == SX:
        return np.array([0.5 + 0.5j, 0.5 - 0.5j, 0.5 - 0.5j, 0.5 + 0.5j], dtype=np.complex128)
    if kind == SY:
        return np.array([0.5 + 0.5j, -0.5 - 0.5j, 0.5 + 0.5j, 0.5 + 0.5j], dtype=np.complex128)
    if kind == CZ:
        m = np.eye(4, dtype=np.complex128)
        m[3, 3] = -1.0
        return m.reshape(-1)
    if kind == SW:
        # sqrt(W), W = (X + Y)/sqrt(2): 1/sqrt2 [[1, -e^{i pi/4}], [e^{-i pi/4}, 1]]
        w = np.exp(1j * math.pi / 4)
        return np.array([s, -s * w, s * np.conj(w), s], dtype=np.complex128)
    if kind == FSIM:
        # fSim(theta = pi/2, phi = pi/6) of the Sycamore RCS experiment
        m = np.zeros((4, 4), dtype=np.complex128)
        m[0, 0] = 1.0
        m[1, 2] = m[2, 1] = -1j
        m[3, 3] = np.exp(-1j * math.pi / 6)
        return m.reshape(-1)
    raise ValueError(f"unknown gate: {kind}")


@dataclass
class Gate:
    kind: str
    qubits: tuple


@dataclass
class Circuit:
    n_qubits: int = 0
    layers: list = field(default_factory=list)


def validate_circuit(c: Circuit) -> None:
    """qcircuit.cpp:32-46."""
    for layer in c.layers:
        touched = set()
        for g in layer:
            want = 2 if g.kind in TWO_QUBIT else 1
            if len(g.qubits) != want:
                raise ValueError("gate has wrong qubit count")
            for q in g.qubits:
                if q < 0 or q >= c.n_qubits:
                    raise ValueError("qubit index out of range")
                if q in touched:
                    raise ValueError("layer gates must act on disjoint qubits")
                touched.add(q)


def cz_pattern(rows: int, cols: int, layer_index: int):
    """qcircuit.cpp:83-102: H0 V0 H1 V1 H2 V2 H3 V3 staggered pairings."""
    p = layer_index % 8
    horizontal = p % 2 == 0
    phase = p // 2
    pairs = []
    if horizontal:
        for r in range(rows):
            for c in range(cols - 1):
                if (c + 2 * (r % 2)) % 4 == phase:
                    pairs.append((r * cols + c, r * cols + c + 1))
    else:
        for r in range(rows - 1):
            for c in range(cols):
                if (r + 2 * (c % 2)) % 4 == phase:
                    pairs.append((r * cols + c, (r + 1) * cols + c))
    return pairs


def rqc_rectangular(rows: int, cols: int, mid_depth: int, seed: int) -> Circuit:
    """qcircuit.cpp:104-140."""
    if rows < 1 or cols < 1 or mid_depth < 0:
        raise ValueError("invalid lattice parameters")
    n = rows * cols
    rng = Rng(seed)
    c = Circuit(n_qubits=n)
    h_layer = [Gate(H, (q,)) for q in range(n)]
    c.layers.append(h_layer)
    last = [-1] * n
    for d in range(mid_depth):
        layer = []
        in_cz = [False] * n
        for a, b in cz_pattern(rows, cols, d):
            layer.append(Gate(CZ, (a, b)))
            in_cz[a] = in_cz[b] = True
        for q in range(n):
            if in_cz[q]:
                continue
            allowed = [g for g in range(3) if g != last[q]]
            pick = allowed[rng.next_below(len(allowed))]
            last[q] = pick
            layer.append(Gate(_SINGLES[pick], (q,)))
        c.layers.append(layer)
    c.layers.append(list(h_layer))
    return c


def _wire(q: int, step: int) -> str:
    return f"w{q}_{step}"


@dataclass
class NetworkSpec:
    """TensorNetwork (network.hpp:17-19): labels, dims and complex64 data per node."""
    labels: list = field(default_factory=list)
    dims: list = field(default_factory=list)
    data: list = field(default_factory=list)
    selector_nodes: list = field(default_factory=list)  # node id of qubit q's <x_q| selector


def gate_data(kind: str) -> np.ndarray:
    """gate_tensor (qcircuit.cpp:63-81): f64 matrix rounded to f32, (out..., in...)."""
    return gate_matrix(kind).astype(np.complex64)


def circuit_to_network(c: Circuit, x) -> NetworkSpec:
    """qcircuit.cpp:142-182: |0> states, one tensor per gate, <x| selectors."""
    validate_circuit(c)
    if len(x) != c.n_qubits:
        raise ValueError("bitstring length does not match circuit")
    net = NetworkSpec()
    step = [0] * c.n_qubits
    for q in range(c.n_qubits):
        net.labels.append([_wire(q, 0)])
        net.dims.append([2])
        net.data.append(np.array([1.0, 0.0], dtype=np.complex64))
    for layer in c.layers:
        for g in layer:
            if g.kind in TWO_QUBIT:
                a, b = g.qubits
                net.labels.append([_wire(a, step[a] + 1), _wire(b, step[b] + 1), _wire(a, step[a]),
                                   _wire(b, step[b])])
                net.dims.append([2, 2, 2, 2])
                step[a] += 1
                step[b] += 1
            else:
                (q,) = g.qubits
                net.labels.append([_wire(q, step[q] + 1), _wire(q, step[q])])
                net.dims.append([2, 2])
                step[q] += 1
            net.data.append(gate_data(g.kind))
    for q in range(c.n_qubits):
        net.selector_nodes.append(len(net.labels))
        net.labels.append([_wire(q, step[q])])
        net.dims.append([2])
        sel = np.zeros(2, dtype=np.complex64)
        sel[1 if x[q] else 0] = 1.0
        net.data.append(sel)
    return net


def bitstrings_for(n_qubits: int, n_bitstrings: int, seed: int):
    """experiments.cpp:185-196: distinct seed-deterministic output strings
    (ascending by value, qubit q = bit q)."""
    rng = Rng(seed ^ 0xC2B2AE3D27D4EB4F)
    space = _M64 if n_qubits >= 63 else (1 << n_qubits)
    want = min(n_bitstrings, space)
    chosen = set()
    while len(chosen) < want:
        chosen.add(rng.next_below(space))
    return [[(v >> q) & 1 for q in range(n_qubits)] for v in sorted(chosen)]


def save_circuit(c: Circuit) -> str:
    """save_circuit text format (qcircuit.cpp:237-247)."""
    out = [f"qubits {c.n_qubits}"]
    for layer in c.layers:
        out.append("layer")
        for g in layer:
            out.append(" ".join([g.kind] + [str(q) for q in g.qubits]))
        out.append("endlayer")
    return "\n".join(out) + "\n"


def load_circuit(text: str) -> Circuit:
    """load_circuit (qcircuit.cpp:249-281)."""
    c = Circuit()
    in_layer = False
    for line in text.splitlines():
        tok = line.split()
        if not tok:
            continue
        if tok[0] == "qubits":
            c.n_qubits = int(tok[1])
        elif tok[0] == "layer":
            c.layers.append([])
            in_layer = True
        elif tok[0] == "endlayer":
            in_layer = False
        else:
            if not in_layer:
                raise ValueError("gate outside layer block")
            if tok[0] not in (H, T, SX, SY, CZ, SW, FSIM):
                raise ValueError("unknown gate: " + tok[0])
            c.layers[-1].append(Gate(tok[0], tuple(int(q) for q in tok[1:])))
    validate_circuit(c)
    return c


# ------------------------------------------------- Sycamore-class (configs[3])
def sycamore_qubits():
    """The 54-site rotated-square layout of the Sycamore chip as grid
    coordinates (row r has the listed column span); site (5, 0) is dropped to
    leave 53 active qubits, as in the RCS experiment.  Qubit index = position
    in this row-major list."""
    spans = [(0, 5, 6), (1, 4, 7), (2, 3, 8), (3, 2, 9), (4, 1, 9), (5, 1, 8), (6, 1, 7),
             (7, 2, 6), (8, 3, 5), (9, 4, 4)]
    sites = []
    for r, c0, c1 in spans:
        for c in range(c0, c1 + 1):
            sites.append((r, c))
    return sites


def sycamore_couplers(sites, pattern: str):
    """Couplers of pattern A/B/C/D: A/B are the two halves of the horizontal
    grid bonds, C/D of the vertical ones (alternating parity), so every qubit
    has at most one coupler per pattern."""
    pos = {s: i for i, s in enumerate(sites)}
    pairs = []
    for (r, c), i in pos.items():
        if pattern in "AB":
            nb = (r, c + 1)
            par = (r + c) % 2 == (0 if pattern == "A" else 1)
        else:
            nb = (r + 1, c)
            par = (r + c) % 2 == (0 if pattern == "C" else 1)
        if par and nb in pos:
            pairs.append((i, pos[nb]))
    return pairs


def sycamore_like(cycles: int, seed: int) -> Circuit:
    """Sycamore-class random circuit: `cycles` cycles of (random single-qubit
    gate from {sqrtX, sqrtY, sqrtW}, never repeating on a qubit) + fSim(pi/2,
    pi/6) on the couplers of the pattern sequence ABCDCDAB, then a final
    single-qubit layer.  Uses the reference Rng for reproducibility."""
    sites = sycamore_qubits()
    n = len(sites)
    rng = Rng(seed)
    c = Circuit(n_qubits=n)
    singles = (SX, SY, SW)
    last = [-1] * n
    order = "ABCDCDAB"

    def single_layer():
        layer = []
        for q in range(n):
            allowed = [g for g in range(3) if g != last[q]]
            pick = allowed[rng.next_below(len(allowed))]
            last[q] = pick
            layer.append(Gate(singles[pick], (q,)))
        return layer

    for cyc in range(cycles):
        c.layers.append(single_layer())
        c.layers.append([Gate(FSIM, pair) for pair in sycamore_couplers(sites, order[cyc % 8])])
    c.layers.append(single_layer())
    return c
