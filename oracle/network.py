"""TEST INFRASTRUCTURE ONLY -- network-level CPU oracle.

Restates the reference's TTGT fold (network.cpp:33-85, :129-177) on top of the C
restatement's dispatch_cgemm (so decisions, log lines and every FP32/FP64 tier
value are the reference's bit for bit), the f64 contraction oracle
(network.cpp:87-110, :141-145, :179-186) and the f64 state-vector oracle
(qcircuit.cpp:197-235).  Small cases only (pure Python around C kernels).
"""
from __future__ import annotations

import numpy as np

from . import make_config, oracle


def _split_pair(la, da, lb, db):
    """network.cpp:33-56"""
    free_a, shared, free_b, fa_d, sh_d, fb_d = [], [], [], [], [], []
    for l, d in zip(la, da):
        if l in lb:
            bd = db[lb.index(l)]
            if bd != d:
                raise ValueError(f"label {l} has extents {d} and {bd}")
            shared.append(l)
            sh_d.append(d)
        else:
            free_a.append(l)
            fa_d.append(d)
    for l, d in zip(lb, db):
        if l not in la:
            free_b.append(l)
            fb_d.append(d)
    return free_a, shared, free_b, fa_d, sh_d, fb_d


def _ttgt(a, b, run_gemm):
    """network.cpp:58-85: permute A to (free_a|shared), B to (shared|free_b), GEMM,
    reinterpret as (free_a|free_b)."""
    (la, da, xa), (lb, db, xb) = a, b
    free_a, shared, free_b, fa_d, sh_d, fb_d = _split_pair(la, da, lb, db)
    ta = np.asarray(xa).reshape(da) if da else np.asarray(xa).reshape(())
    tb = np.asarray(xb).reshape(db) if db else np.asarray(xb).reshape(())
    pa = np.ascontiguousarray(np.transpose(ta, [la.index(l) for l in free_a + shared]))
    pb = np.ascontiguousarray(np.transpose(tb, [lb.index(l) for l in shared + free_b]))
    m = int(np.prod(fa_d)) if fa_d else 1
    k = int(np.prod(sh_d)) if sh_d else 1
    n = int(np.prod(fb_d)) if fb_d else 1
    c = run_gemm(pa.reshape(m, k), pb.reshape(k, n))
    return free_a + free_b, fa_d + fb_d, np.asarray(c).reshape(-1)


def _fold(nodes, path, contract):
    """network.cpp:149-168 fold_path (SSA ids)."""
    if not nodes:
        raise ValueError("empty network")
    live = {i: t for i, t in enumerate(nodes)}
    nxt = len(nodes)
    for ia, ib in path:
        if ia == ib or ia not in live or ib not in live:
            raise ValueError("step references a dead or unknown node")
        r = contract(live[ia], live[ib])
        del live[ia]
        del live[ib]
        live[nxt] = r
        nxt += 1
    if len(live) != 1:
        raise ValueError("path leaves more than one node")
    return next(iter(live.values()))


def contract_network(spec, path, cfg=None):
    """contract_network (network.cpp:172-177) with the C restatement's dispatch.
    Returns (labels, dims, complex64 data, decision-log lines)."""
    o = oracle()
    cfg = cfg if cfg is not None else make_config()
    lines = []

    def gemm(ma, mb):
        rc, c, res = o.dispatch_cgemm(ma.astype(np.complex64), mb.astype(np.complex64), cfg)
        if rc:
            raise RuntimeError(f"oracle dispatch failed rc={rc}")
        lines.append(res.line.decode())
        return c

    nodes = [(list(l), list(d), np.asarray(x, dtype=np.complex64))
             for l, d, x in zip(spec.labels, spec.dims, spec.data)]
    labels, dims, data = _fold(nodes, path, lambda a, b: _ttgt(a, b, gemm))
    return labels, dims, data.astype(np.complex64), lines


def contract_network_f64(spec, path):
    """contract_network_oracle (network.cpp:179-186): everything in f64."""
    nodes = [(list(l), list(d), np.asarray(x, dtype=np.complex128))
             for l, d, x in zip(spec.labels, spec.dims, spec.data)]
    return _fold(nodes, path, lambda a, b: _ttgt(a, b, lambda x, y: x @ y))


def statevector(circuit):
    """statevector_oracle (qcircuit.cpp:197-225): qubit q = bit q of the index."""
    from paper_2303_08989_b200.circuits import CZ, FSIM, gate_matrix  # workload definition only
    n = circuit.n_qubits
    if n > 24:
        raise ValueError("state-vector oracle limited to 24 qubits")
    state = np.zeros(1 << n, dtype=np.complex128)
    state[0] = 1.0
    idx = np.arange(1 << n)
    for layer in circuit.layers:
        for g in layer:
            if g.kind == CZ:
                ma, mb = 1 << g.qubits[0], 1 << g.qubits[1]
                sel = (idx & ma != 0) & (idx & mb != 0)
                state[sel] = -state[sel]
                continue
            if g.kind == FSIM:
                # generic two-qubit unitary, index bits (q_a, q_b) = row-major (oa, ob)
                u = gate_matrix(g.kind).reshape(4, 4)
                ma, mb = 1 << g.qubits[0], 1 << g.qubits[1]
                base = idx[((idx & ma) == 0) & ((idx & mb) == 0)]
                cols = [base, base | mb, base | ma, base | ma | mb]
                vals = [state[c].copy() for c in cols]
                for r in range(4):
                    state[cols[r]] = sum(u[r, cc] * vals[cc] for cc in range(4))
                continue
            u = gate_matrix(g.kind)
            mq = 1 << g.qubits[0]
            lo = idx[(idx & mq) == 0]
            a0 = state[lo].copy()
            a1 = state[lo | mq].copy()
            state[lo] = u[0] * a0 + u[1] * a1
            state[lo | mq] = u[2] * a0 + u[3] * a1
    return state


def amplitude_sv(circuit, x):
    """amplitude_oracle (qcircuit.cpp:227-235)."""
    st = statevector(circuit)
    i = sum(1 << q for q, b in enumerate(x) if b)
    return st[i]


def greedy_path(spec):
    """greedy_path (network.cpp:204-315), pure Python, for planning-logic checks."""
    live = [(i, list(l), list(d)) for i, (l, d) in enumerate(zip(spec.labels, spec.dims))]
    nxt = len(live)
    steps = []
    while len(live) > 1:
        best = None
        for adjacent_only in (True, False):
            for x in range(len(live)):
                for y in range(x + 1, len(live)):
                    ix, lx, dx = live[x]
                    iy, ly, dy = live[y]
                    adj = any(l in ly for l in lx)
                    if adjacent_only and not adj:
                        continue
                    if adjacent_only:
                        fx = int(np.prod([d for l, d in zip(lx, dx) if l not in ly])) if lx else 1
                        fy = int(np.prod([d for l, d in zip(ly, dy) if l not in lx])) if ly else 1
                        size = fx * fy
                    else:
                        size = int(np.prod(dx + dy)) if dx + dy else 1
                    ids = (min(ix, iy), max(ix, iy))
                    if best is None or size < best[0] or (size == best[0] and ids < best[1]):
                        best = (size, ids, x, y)
            if best is not None:
                break
        _, ids, x, y = best
        ix, lx, dx = live[x]
        iy, ly, dy = live[y]
        ml = [l for l in lx if l not in ly] + [l for l in ly if l not in lx]
        md = [d for l, d in zip(lx, dx) if l not in ly] + [d for l, d in zip(ly, dy) if l not in lx]
        steps.append(ids)
        for j in sorted((x, y), reverse=True):
            del live[j]
        live.append((nxt, ml, md))
        nxt += 1
    return steps
