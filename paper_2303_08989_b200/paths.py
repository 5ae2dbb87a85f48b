"""Contraction-path search beyond the reference's greedy_path.

The reference's greedy (network.cpp:204-315) minimizes only the size of each
pairwise result; on Sycamore-class circuits its intermediates explode (2^34
elements at 8 cycles, 2^85 at 12).  `random_greedy_path` is a randomized
greedy in the opt_einsum style: the score of contracting adjacent tensors a, b
is size(a.b) - size(a) - size(b) (how much memory the step frees), perturbed
by Boltzmann noise; many trials are run and the path with the lowest flop
count whose largest intermediate fits `max_width` (log2 elements) wins.
Paths use the reference's SSA numbering (network.hpp:22-26) and feed the same
device executor.
"""
from __future__ import annotations

import heapq
import math
import random

import numpy as np

from .circuits import NetworkSpec


def _log2size(dims):
    return sum(math.log2(d) for d in dims)


def _trial(labels, dims_of, rng: random.Random, temperature: float):
    """One randomized greedy pass.  labels: list of label tuples per node."""
    live = {i: tuple(ls) for i, ls in enumerate(labels)}
    where = {}
    for i, ls in live.items():
        for l in ls:
            where.setdefault(l, set()).add(i)
    nxt = len(labels)

    def size(ls):
        s = 1
        for l in ls:
            s *= dims_of[l]
        return s

    def merged(a, b):
        sa, sb = set(live[a]), set(live[b])
        return tuple([l for l in live[a] if l not in sb] + [l for l in live[b] if l not in sa])

    def score(a, b):
        out = merged(a, b)
        s = size(out) - size(live[a]) - size(live[b])
        if temperature > 0:
            g = -math.log(-math.log(rng.random() + 1e-300))  # Gumbel noise
            s -= temperature * g * max(size(live[a]), size(live[b]))
        return s

    heap = []
    for l, owners in where.items():
        if len(owners) == 2:
            a, b = sorted(owners)
            heapq.heappush(heap, (score(a, b), a, b))
    steps, flops, width = [], 0.0, 0.0
    while len(live) > 1:
        while heap:
            sc, a, b = heapq.heappop(heap)
            if a in live and b in live:
                break
        else:
            # disconnected: outer product of the two smallest
            a, b = sorted(live, key=lambda i: size(live[i]))[:2]
        out = merged(a, b)
        sa = set(live[a])
        k = 1
        for l in live[b]:
            if l in sa:
                k *= dims_of[l]
        flops += 8.0 * size(out) * k
        width = max(width, _log2size([dims_of[l] for l in out]))
        steps.append((min(a, b), max(a, b)))
        for l in live[a]:
            where[l].discard(a)
        for l in live[b]:
            where[l].discard(b)
        del live[a]
        del live[b]
        live[nxt] = out
        for l in out:
            where[l].add(nxt)
        neigh = set()
        for l in out:
            neigh |= where[l]
        neigh.discard(nxt)
        for o in neigh:
            heapq.heappush(heap, (score(min(o, nxt), max(o, nxt)), min(o, nxt), max(o, nxt)))
        nxt += 1
    return steps, flops, width


def random_greedy_path(spec: NetworkSpec, trials: int = 64, max_width: float = 30.0,
                       temperatures=(0.0, 0.01, 0.03, 0.1, 0.3), seed: int = 0):
    """Best-of-trials randomized greedy: returns (path, flops, log2 width)."""
    dims_of = {}
    for ls, ds in zip(spec.labels, spec.dims):
        for l, d in zip(ls, ds):
            dims_of[l] = d
    rng = random.Random(seed)
    best = None
    for t in range(trials):
        temp = temperatures[t % len(temperatures)]
        steps, flops, width = _trial(spec.labels, dims_of, rng, temp)
        key = (width > max_width, flops if width <= max_width else width)
        if best is None or key < best[0]:
            best = (key, steps, flops, width)
    return best[1], best[2], best[3]


def bisection_path(spec: NetworkSpec, trials: int = 8, leaf: int = 12, seed: int = 0,
                   max_width: float = 30.0):
    """Recursive Kernighan-Lin bisection of the tensor graph (edge weight =
    log2 bond dimension): every subtree is contracted before its sibling, so
    a subtree's intermediate is exactly its cut; leaves (<= `leaf` tensors)
    are ordered by the randomized greedy.  Best of `trials` seeds."""
    import networkx as nx
    from networkx.algorithms.community import kernighan_lin_bisection

    dims_of, owners = {}, {}
    for i, (ls, ds) in enumerate(zip(spec.labels, spec.dims)):
        for l, d in zip(ls, ds):
            dims_of[l] = d
            owners.setdefault(l, []).append(i)
    g = nx.Graph()
    g.add_nodes_from(range(len(spec.labels)))
    for l, own in owners.items():
        if len(own) == 2:
            a, b = own
            w = math.log2(dims_of[l])
            if g.has_edge(a, b):
                g[a][b]["weight"] += w
            else:
                g.add_edge(a, b, weight=w)

    best = None
    for t in range(trials):
        rng = random.Random(seed + 7919 * t)

        def split(nodes):
            if len(nodes) <= leaf:
                return list(nodes)
            sub = g.subgraph(nodes)
            comps = list(nx.connected_components(sub))
            if len(comps) > 1:
                comps.sort(key=len)
                a = set(comps[0])
                b = set(nodes) - a
            else:
                a, b = kernighan_lin_bisection(sub, weight="weight", seed=rng.randrange(1 << 30))
            return [split(sorted(a)), split(sorted(b))]

        tree = split(list(range(len(spec.labels))))
        # post-order -> SSA steps; leaves (lists of ints) by a local greedy
        live_labels = {i: list(ls) for i, ls in enumerate(spec.labels)}
        counter = [len(spec.labels)]
        steps = []

        def contract(a, b):
            la, lb = live_labels.pop(a), live_labels.pop(b)
            sa, sb = set(la), set(lb)
            live_labels[counter[0]] = [l for l in la if l not in sb] + [l for l in lb if l not in sa]
            steps.append((min(a, b), max(a, b)))
            counter[0] += 1
            return counter[0] - 1

        def leaf_order(ids):
            ids = list(ids)
            while len(ids) > 1:
                bestp = None
                for x in range(len(ids)):
                    for y in range(x + 1, len(ids)):
                        la, lb = live_labels[ids[x]], live_labels[ids[y]]
                        shared = set(la) & set(lb)
                        out = _log2size([dims_of[l] for l in la if l not in shared] +
                                        [dims_of[l] for l in lb if l not in shared])
                        key = (not shared, out + rng.random() * 1e-3)
                        if bestp is None or key < bestp[0]:
                            bestp = (key, x, y)
                _, x, y = bestp
                nid = contract(ids[x], ids[y])
                ids = [i for j, i in enumerate(ids) if j not in (x, y)] + [nid]
            return ids[0]

        def walk(node):
            if node and isinstance(node[0], list):
                left = walk(node[0])
                right = walk(node[1])
                return contract(left, right)
            if isinstance(node, list) and node and isinstance(node[0], int):
                return leaf_order(node)
            return walk(node[0])

        walk(tree)
        flops, width = path_cost(spec, steps)
        key = (width > max_width, flops if width <= max_width else width)
        if best is None or key < best[0]:
            best = (key, steps, flops, width)
    return best[1], best[2], best[3]


def path_cost(spec: NetworkSpec, path):
    """(flops, log2 of the largest intermediate) of an SSA path."""
    dims_of = {}
    for ls, ds in zip(spec.labels, spec.dims):
        for l, d in zip(ls, ds):
            dims_of[l] = d
    live = {i: list(ls) for i, ls in enumerate(spec.labels)}
    nxt = len(spec.labels)
    flops, width = 0.0, 0.0
    for a, b in path:
        la, lb = live.pop(a), live.pop(b)
        sb, sa = set(lb), set(la)
        out = [l for l in la if l not in sb] + [l for l in lb if l not in sa]
        k = float(np.prod([dims_of[l] for l in la if l in sb])) if la else 1.0
        flops += 8.0 * float(np.prod([dims_of[l] for l in out]) if out else 1.0) * k
        width = max(width, _log2size([dims_of[l] for l in out]))
        live[nxt] = out
        nxt += 1
    return flops, width
