"""Sliced contraction: slice finder, slice scheduler and the cross-GPU sum.

Slicing a set S of bond labels turns one contraction into
prod(dims(S)) independent sub-contractions whose values sum to the original.
Every slice has the same node set, SSA path and shapes, so one device plan /
captured CUDA graph serves all of them and only the nodes touching S change
data.  Slices are the data-parallel unit: rank r of W evaluates slice ids
r, r+W, r+2W, ... with no data-path communication, then ONE collective
(all_gather of the per-slice complex values, 8 bytes each) lets every rank sum
them in slice order in float64 -- so the amplitude is bit-identical for any
number of GPUs.

The reference has no slicing; this is the B200 build's
multi-GPU layer (BASELINE.json configs[3]).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .circuits import NetworkSpec


def intermediates(spec: NetworkSpec, path, drop=()):
    """(labels, dims) of every step result along the SSA path (network.cpp:149-168),
    with the labels in `drop` removed (sliced)."""
    drop = set(drop)
    live = {}
    for i, (ls, ds) in enumerate(zip(spec.labels, spec.dims)):
        live[i] = [(l, d) for l, d in zip(ls, ds) if l not in drop]
    nxt = len(spec.labels)
    out = []
    for ia, ib in path:
        a, b = live.pop(ia), live.pop(ib)
        la = {l for l, _ in a}
        lb = {l for l, _ in b}
        res = [(l, d) for l, d in a if l not in lb] + [(l, d) for l, d in b if l not in la]
        live[nxt] = res
        nxt += 1
        out.append(res)
    return out


def _size(t):
    s = 1
    for _, d in t:
        s *= d
    return s


def contraction_cost(spec: NetworkSpec, path, drop=()):
    """(max intermediate elements, total complex MACs) of the path."""
    drop = set(drop)
    live = {i: [(l, d) for l, d in zip(ls, ds) if l not in drop]
            for i, (ls, ds) in enumerate(zip(spec.labels, spec.dims))}
    nxt = len(spec.labels)
    biggest, macs = 1, 0
    for ia, ib in path:
        a, b = live.pop(ia), live.pop(ib)
        la = {l for l, _ in a}
        lb = {l for l, _ in b}
        m = _size([(l, d) for l, d in a if l not in lb])
        n = _size([(l, d) for l, d in b if l not in la])
        k = _size([(l, d) for l, d in a if l in lb])
        macs += m * n * k
        res = [(l, d) for l, d in a if l not in lb] + [(l, d) for l, d in b if l not in la]
        biggest = max(biggest, _size(res))
        live[nxt] = res
        nxt += 1
    return biggest, macs


def find_slices(spec: NetworkSpec, path, n_labels: int | None = None, max_elems: int | None = None):
    """Greedy slice finder: repeatedly slice the bond that appears in the
    largest intermediates (weighted by size) until `n_labels` bonds are sliced
    or the largest intermediate is <= max_elems.  Deterministic (ties by name)."""
    count = {}
    for ls in spec.labels:
        for l in ls:
            count[l] = count.get(l, 0) + 1
    bonds = sorted(l for l, c in count.items() if c == 2)
    sliced = []
    while True:
        inter = intermediates(spec, path, sliced)
        biggest = max((_size(t) for t in inter), default=1)
        if n_labels is not None and len(sliced) >= n_labels:
            break
        if n_labels is None and max_elems is not None and biggest <= max_elems:
            break
        score = {}
        for t in inter:
            s = _size(t)
            for l, _ in t:
                if l in count and count[l] == 2 and l not in sliced:
                    score[l] = score.get(l, 0) + s
        cands = [l for l in bonds if l in score and l not in sliced]
        if not cands:
            break
        best = max(cands, key=lambda l: (score[l], [-ord(ch) for ch in l]))
        sliced.append(best)
    return sliced


def label_dims(spec: NetworkSpec):
    out = {}
    for ls, ds in zip(spec.labels, spec.dims):
        for l, d in zip(ls, ds):
            out[l] = d
    return out


def assignment(slice_id: int, dims):
    """Mixed-radix digits of slice_id (last label fastest)."""
    digits = []
    for d in reversed(dims):
        digits.append(slice_id % d)
        slice_id //= d
    return list(reversed(digits))


def slice_spec(spec: NetworkSpec, sliced, values) -> NetworkSpec:
    """The sub-network with label sliced[i] fixed to values[i] in both endpoints."""
    fix = dict(zip(sliced, values))
    out = NetworkSpec(selector_nodes=list(spec.selector_nodes))
    for ls, ds, x in zip(spec.labels, spec.dims, spec.data):
        t = np.asarray(x, dtype=np.complex64).reshape(ds) if ds else np.asarray(x).reshape(())
        idx = tuple(fix[l] if l in fix else slice(None) for l in ls)
        t = t[idx] if ls else t
        out.labels.append([l for l in ls if l not in fix])
        out.dims.append([d for l, d in zip(ls, ds) if l not in fix])
        out.data.append(np.ascontiguousarray(t).reshape(-1))
    return out


def var_nodes(spec: NetworkSpec, sliced):
    s = set(sliced)
    return [i for i, ls in enumerate(spec.labels) if s.intersection(ls)]


def rank_slices(n_slices: int, rank: int, world: int):
    """Static round-robin: all slices cost the same (identical path and shapes)."""
    return list(range(rank, n_slices, world))


@dataclass
class SlicePlan:
    spec: NetworkSpec
    path: list
    sliced: list
    dims: list
    n_slices: int
    var: list
    base: NetworkSpec  # slice 0 (shapes of every slice)

    @classmethod
    def build(cls, spec: NetworkSpec, path, sliced):
        dims_all = label_dims(spec)
        dims = [dims_all[l] for l in sliced]
        n = int(np.prod(dims)) if dims else 1
        base = slice_spec(spec, sliced, [0] * len(sliced))
        return cls(spec, list(path), list(sliced), dims, n, var_nodes(spec, sliced), base)

    def run_data(self, slice_id: int):
        """Data of the variable nodes for one slice (the same arrays slice_spec
        gives them; only the variable nodes are sliced -- fixing the labels of
        all ~1000 nodes per slice cost 1.7 ms of host time per slice)."""
        fix = dict(zip(self.sliced, assignment(slice_id, self.dims)))
        out = []
        for i in self.var:
            ls, ds = self.spec.labels[i], self.spec.dims[i]
            t = np.asarray(self.spec.data[i], dtype=np.complex64).reshape(ds)
            t = t[tuple(fix[l] if l in fix else slice(None) for l in ls)]
            out.append(np.ascontiguousarray(t).reshape(-1))
        return out


def ordered_sum(values_by_slice) -> complex:
    """float64 sum in slice order (reproducible for any world size)."""
    acc = 0j
    for v in values_by_slice:
        acc += complex(v)
    return acc


def gather_slice_values(local_ids, local_vals, n_slices: int, world: int, group=None):
    """One collective: all_gather the per-slice complex64 values; returns the
    full slice-ordered vector on every rank."""
    if world == 1:
        out = np.zeros(n_slices, np.complex64)
        out[np.asarray(local_ids, dtype=np.int64)] = local_vals
        return out
    import torch
    import torch.distributed as dist
    per = (n_slices + world - 1) // world
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    buf = torch.zeros(per, 2, dtype=torch.float32, device=dev)
    lv = np.asarray(local_vals, dtype=np.complex64).view(np.float32).reshape(-1, 2)
    buf[: len(local_ids)] = torch.from_numpy(lv.copy()).to(dev)
    outs = [torch.zeros_like(buf) for _ in range(world)]
    dist.all_gather(outs, buf, group=group)
    full = np.zeros(n_slices, np.complex64)
    for r, t in enumerate(outs):
        ids = rank_slices(n_slices, r, world)
        vals = t.cpu().numpy().view(np.complex64).reshape(-1)[: len(ids)]
        full[np.asarray(ids, dtype=np.int64)] = vals
    return full


def sliced_amplitude(evaluate, plan: SlicePlan, rank: int = 0, world: int = 1, group=None):
    """evaluate(list_of_slice_ids) -> complex64 values (device batch or oracle).
    Returns (amplitude, full per-slice vector)."""
    ids = rank_slices(plan.n_slices, rank, world)
    vals = evaluate(ids) if ids else np.zeros(0, np.complex64)
    full = gather_slice_values(ids, vals, plan.n_slices, world, group)
    return ordered_sum(full), full


def device_evaluator(network, plan: SlicePlan, config=None, chunk: int = 64):
    """Evaluate slices on the GPU: one plan / graph, variable-node data per slice."""
    def evaluate(ids):
        out = []
        for c0 in range(0, len(ids), chunk):
            runs = [plan.run_data(i) for i in ids[c0:c0 + chunk]]
            out.append(network.node_batch(plan.path, plan.var, runs, config))
        return np.concatenate(out) if out else np.zeros(0, np.complex64)
    return evaluate


__all__ = ["intermediates", "contraction_cost", "find_slices", "slice_spec", "SlicePlan",
           "rank_slices", "ordered_sum", "gather_slice_values", "sliced_amplitude",
           "device_evaluator", "assignment"]
