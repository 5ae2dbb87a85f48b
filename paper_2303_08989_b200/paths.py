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


def _tensor_graph(spec: NetworkSpec):
    """Graph of the network: nodes = tensors, edge weight = sum of log2 bond dims."""
    import networkx as nx
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
    return g, dims_of


def _spectral_split(sub, rng: random.Random, imbalance):
    """Two-way cut of a connected graph: nodes ordered by the Fiedler vector,
    cut at the cheapest position inside a randomly placed window (sampled
    imbalance), refined by Kernighan-Lin swaps (sizes preserved)."""
    import networkx as nx
    from networkx.algorithms.community import kernighan_lin_bisection
    nodes = list(sub.nodes)
    n = len(nodes)
    try:
        fv = nx.fiedler_vector(sub, weight="weight", normalized=True, method="tracemin_lu",
                               seed=rng.randrange(1 << 30))
        order = [nodes[i] for i in np.argsort(fv, kind="stable")]
    except Exception:  # tiny or degenerate graphs
        order = list(nodes)
        rng.shuffle(order)
    lo, hi = imbalance
    f = rng.uniform(lo, hi)
    w0, w1 = max(1, int((f - 0.08) * n)), min(n - 1, int((f + 0.08) * n))
    side = {}
    cut, best = 0.0, None
    for pos, v in enumerate(order[:-1]):
        side[v] = 0
        for u, d in sub[v].items():
            cut += -d["weight"] if side.get(u) == 0 else d["weight"]
        if w0 <= pos + 1 <= w1 and (best is None or cut < best[0]):
            best = (cut, pos + 1)
    k = best[1] if best else max(1, n // 2)
    a, b = set(order[:k]), set(order[k:])
    if n > 4:
        a, b = kernighan_lin_bisection(sub, partition=(a, b), max_iter=4, weight="weight",
                                       seed=rng.randrange(1 << 30))
    return a, b


def partition_path(spec: NetworkSpec, trials: int = 16, leaf: int = 10, seed: int = 0,
                   max_width: float = 30.0, imbalance=(0.3, 0.7)):
    """Divisive contraction tree (the hyper-optimized recipe of Gray & Kourtis,
    with a spectral + Kernighan-Lin graph partitioner instead of a hypergraph
    one): recursively cut the tensor graph in two (Fiedler-vector order,
    cheapest cut inside a randomly sampled imbalance window, KL refinement);
    every subtree is contracted before its sibling, so an intermediate is the
    boundary of its part.  Parts of <= `leaf` tensors are ordered by a local
    greedy.  Best of `trials` samples (lowest flops among widths <= max_width,
    else lowest width).  Returns (path, flops, log2 width)."""
    import networkx as nx
    g, dims_of = _tensor_graph(spec)

    best = None
    for t in range(trials):
        rng = random.Random(seed + 7919 * t)

        def split(nodes):
            if len(nodes) <= leaf:
                return list(nodes)
            sub = g.subgraph(nodes)
            comps = sorted(nx.connected_components(sub), key=len)
            if len(comps) > 1:
                a = set(comps[0])
                b = set(nodes) - a
            else:
                a, b = _spectral_split(sub, rng, imbalance)
            if not a or not b:
                half = len(nodes) // 2
                a, b = set(list(nodes)[:half]), set(list(nodes)[half:])
            return [split(sorted(a)), split(sorted(b))]

        tree = split(list(range(len(spec.labels))))
        steps = _tree_to_steps(spec, tree, dims_of, rng)
        flops, width = path_cost(spec, steps)
        key = (width > max_width, flops if width <= max_width else width)
        if best is None or key < best[0]:
            best = (key, steps, flops, width)
    return best[1], best[2], best[3]


def _tree_to_steps(spec, tree, dims_of, rng):
    """Post-order SSA steps of a nested-list contraction tree; leaf groups
    (lists of tensor ids) are ordered by the smallest-result greedy."""
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
        return leaf_order(node)

    walk(tree)
    return steps


def path_cost(spec: NetworkSpec, path):
    """(flops, log2 of the largest intermediate) of an SSA path (float
    arithmetic: no integer overflow on hopeless paths)."""
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
        lk = _log2size([dims_of[l] for l in la if l in sb])
        lo = _log2size([dims_of[l] for l in out])
        flops += 8.0 * 2.0 ** (lo + lk)
        width = max(width, lo)
        live[nxt] = out
        nxt += 1
    return flops, width


def presimplify(spec: NetworkSpec):
    """Absorb every tensor of rank <= 2 (single-qubit gates, |0> states, <x|
    selectors) into a neighbour until none is left -- the contractions never
    grow a tensor, so they are free in width.  Returns (steps, ids, reduced):
    the SSA steps taken, the SSA id of every surviving tensor, and a
    NetworkSpec (labels/dims only) of the reduced network."""
    live = {i: list(ls) for i, ls in enumerate(spec.labels)}
    dims_of = {}
    for ls, ds in zip(spec.labels, spec.dims):
        for l, d in zip(ls, ds):
            dims_of[l] = d
    holder = {}
    for i, ls in live.items():
        for l in ls:
            holder.setdefault(l, set()).add(i)
    nxt = len(spec.labels)
    steps = []
    changed = True
    while changed and len(live) > 1:
        changed = False
        for i in sorted(live):
            if i not in live or len(live[i]) > 2:
                continue
            nbs = sorted({h for l in live[i] for h in holder[l] if h != i and h in live})
            if not nbs:
                continue
            # the neighbour sharing the most bonds (the result is never larger than it)
            j = max(nbs, key=lambda h: (len(set(live[h]) & set(live[i])), -h))
            la, lb = live.pop(min(i, j)), live.pop(max(i, j))
            sa, sb = set(la), set(lb)
            out = [l for l in la if l not in sb] + [l for l in lb if l not in sa]
            for l in la:
                holder[l].discard(min(i, j))
            for l in lb:
                holder[l].discard(max(i, j))
            live[nxt] = out
            for l in out:
                holder[l].add(nxt)
            steps.append((min(i, j), max(i, j)))
            nxt += 1
            changed = True
    ids = sorted(live)
    reduced = NetworkSpec(labels=[list(live[i]) for i in ids],
                          dims=[[dims_of[l] for l in live[i]] for i in ids], data=[])
    return steps, ids, reduced


def remap_path(steps_pre, ids, n_orig, reduced_path):
    """Compose presimplify's steps with a path over the reduced network into
    one SSA path over the original network."""
    n_red = len(ids)
    ssa = {r: ids[r] for r in range(n_red)}
    nxt = n_orig + len(steps_pre)
    out = list(steps_pre)
    for r, (a, b) in enumerate(reduced_path):
        x, y = ssa[a], ssa[b]
        out.append((min(x, y), max(x, y)))
        ssa[n_red + r] = nxt
        nxt += 1
    return out


def reconfigure_path(spec: NetworkSpec, path, k: int = 8, passes: int = 3, seed: int = 0,
                     latency_macs: float = 1e4, time_model: bool = False, native: bool = True):
    """Subtree reconfiguration; the native C++ engine (tcec_path_reconfigure,
    csrc/path_search.cu) unless native=False (the Python reference below)."""
    if native:
        return _reconfigure_native(spec, path, k, passes, seed, latency_macs, time_model)
    return _reconfigure_py(spec, path, k, passes, seed, latency_macs, time_model)


def _reconfigure_native(spec, path, k, passes, seed, latency_macs, time_model):
    import ctypes as C
    from ._lib import check, load
    lib = load()
    names = {}
    ranks, labels, dims = [], [], []
    for ls, ds in zip(spec.labels, spec.dims):
        ranks.append(len(ls))
        for l, d in zip(ls, ds):
            labels.append(names.setdefault(l, len(names)))
            dims.append(int(d))
    n = len(spec.labels)
    flat = [x for st in path for x in st]
    out = (C.c_int * max(len(flat), 1))()
    check(lib.tcec_path_reconfigure(
        n, (C.c_int * max(n, 1))(*ranks), (C.c_int * max(len(labels), 1))(*labels),
        (C.c_int64 * max(len(dims), 1))(*dims), (C.c_int * max(len(flat), 1))(*flat), len(path),
        int(k), int(passes), int(bool(time_model)), float(latency_macs), int(seed) & (2 ** 64 - 1), out))
    steps = [(out[2 * i], out[2 * i + 1]) for i in range(len(path))]
    f, w = path_cost(spec, steps)
    return steps, f, w


def _reconfigure_py(spec: NetworkSpec, path, k: int = 8, passes: int = 3, seed: int = 0,
                    latency_macs: float = 1e4, time_model: bool = False):
    """Subtree reconfiguration (cotengra's `subtree_reconfigure`): for every
    node of the contraction tree take a frontier of up to `k` sub-pieces and
    replace the way they are combined by the cheapest order (dynamic
    programming over subsets).  In a closed network every bond joins exactly
    two tensors, so the open legs of a union of pieces are the XOR of their
    leg bitmasks.  `time_model` scores a step by its estimated B200 time
    (tensor-core tiers faster, HBM floor) instead of its MACs.  Step cost = m n k MACs, plus `latency_macs` per element of
    k when the step has < 65536 outputs: the FP32 tier must add each output's
    k products in one sequential RN chain (kernels_scalar.cpp:76-87), so a
    few-output, long-k step is bound by FADD latency (~4 ns per add, about
    1e4 MACs of throughput), not by its flops.  Returns (path, flops, log2 width)."""
    rng = random.Random(seed)
    bit, lw = {}, []
    for ls, ds in zip(spec.labels, spec.dims):
        for l, d in zip(ls, ds):
            if l not in bit:
                bit[l] = len(lw)
                lw.append(math.log2(d))
    uniform = all(w == 1.0 for w in lw)

    def width(mask):
        if uniform:
            return float(mask.bit_count())
        w, i = 0.0, 0
        while mask:
            if mask & 1:
                w += lw[i]
            mask >>= 1
            i += 1
        return w

    n = len(spec.labels)
    # tree nodes: id -> (left, right) for internal; leaves are ids < n
    legs = {}
    for i, ls in enumerate(spec.labels):
        m = 0
        for l in ls:
            m |= 1 << bit[l]
        legs[i] = m
    children = {}
    nxt = n
    for a, b in path:
        children[nxt] = (a, b)
        legs[nxt] = legs[a] ^ legs[b]
        nxt += 1
    root = nxt - 1

    def step_cost(ma, mb):
        return model_step_cost(width(ma), width(mb), width(ma ^ mb), time_model, latency_macs)

    def optimize(node):
        """Reconfigure the top of the subtree at `node`; True if improved."""
        nonlocal nxt
        if node not in children:
            return False
        frontier = [node]
        internal_top = []
        while len(frontier) < k:
            cand = [p for p in frontier if p in children]
            if not cand:
                break
            p = max(cand, key=lambda q: (width(legs[q]), rng.random()))
            frontier.remove(p)
            internal_top.append(p)
            frontier.extend(children[p])
        if len(frontier) < 3:
            return False
        old = sum(step_cost(legs[children[p][0]], legs[children[p][1]]) for p in internal_top)
        K = len(frontier)
        pm = [legs[p] for p in frontier]
        full = (1 << K) - 1
        sub_legs = [0] * (full + 1)
        for s in range(1, full + 1):
            low = s & -s
            sub_legs[s] = sub_legs[s ^ low] ^ pm[low.bit_length() - 1]
        cost = [0.0] * (full + 1)
        choice = [0] * (full + 1)
        order = sorted(range(1, full + 1), key=lambda s: s.bit_count())
        for s in order:
            if s & (s - 1) == 0:
                continue
            low = s & -s
            best_c, best_a = None, 0
            a = (s - 1) & s
            while a:
                if a & low:
                    b = s ^ a
                    c = cost[a] + cost[b] + step_cost(sub_legs[a], sub_legs[b])
                    if best_c is None or c < best_c:
                        best_c, best_a = c, a
                a = (a - 1) & s
            cost[s], choice[s] = best_c, best_a
        if cost[full] >= old * (1 - 1e-9):
            return False

        # rebuild: the DP tree replaces internal_top; the root keeps its id
        def build(s, node_id=None):
            if s & (s - 1) == 0:
                return frontier[s.bit_length() - 1]
            nonlocal nxt
            a = choice[s]
            l, r = build(a), build(s ^ a)
            if node_id is None:
                node_id = nxt
                nxt += 1
            children[node_id] = (l, r)
            legs[node_id] = legs[l] ^ legs[r]
            return node_id

        for p in internal_top:
            if p != node:
                del children[p]
        build(full, node)
        return True

    for _ in range(passes):
        improved = False
        stack, order_nodes = [root], []
        while stack:
            x = stack.pop()
            if x in children:
                order_nodes.append(x)
                stack.extend(children[x])
        for x in reversed(order_nodes):   # bottom-up
            if x in children:
                improved |= optimize(x)
        if not improved:
            break

    # tree -> SSA steps (post-order)
    steps, ssa = [], {}
    cnt = [n]

    def emit(x):
        if x < n:
            return x
        l, r = children[x]
        a, b = emit(l), emit(r)
        steps.append((min(a, b), max(a, b)))
        cnt[0] += 1
        return cnt[0] - 1

    import sys
    old_lim = sys.getrecursionlimit()
    sys.setrecursionlimit(max(old_lim, 10000))
    try:
        emit(root)
    finally:
        sys.setrecursionlimit(old_lim)
    flops, w = path_cost(spec, steps)
    return steps, flops, w


def _drop_labels(spec: NetworkSpec, drop) -> NetworkSpec:
    drop = set(drop)
    return NetworkSpec(labels=[[l for l in ls if l not in drop] for ls in spec.labels],
                       dims=[[d for l, d in zip(ls, ds) if l not in drop]
                             for ls, ds in zip(spec.labels, spec.dims)], data=[])


def _sliced_cost(spec: NetworkSpec, path, drop):
    """(total flops over all slices, log2 per-slice width) with `drop` sliced."""
    dims_of = {}
    for ls, ds in zip(spec.labels, spec.dims):
        for l, d in zip(ls, ds):
            dims_of[l] = d
    f, w = path_cost(_drop_labels(spec, drop), path)
    return f * float(np.prod([dims_of[l] for l in drop])) if drop else f, w


def find_slices_exact(spec: NetworkSpec, path, max_log2: float, candidates: int = 32,
                      time_model: bool = False):
    """Greedy slicer with exact evaluation: among the bonds of the currently
    largest intermediates, slice the one that minimises the total flops over
    all slices, until the per-slice width is <= max_log2."""
    count = {}
    for ls in spec.labels:
        for l in ls:
            count[l] = count.get(l, 0) + 1
    sliced = []
    while True:
        red = _drop_labels(spec, sliced)
        live = {i: list(ls) for i, ls in enumerate(red.labels)}
        dims_of = {l: d for ls, ds in zip(spec.labels, spec.dims) for l, d in zip(ls, ds)}
        nxt = len(red.labels)
        inter = []
        for a, b in path:
            la, lb = live.pop(a), live.pop(b)
            sa, sb = set(la), set(lb)
            out = [l for l in la if l not in sb] + [l for l in lb if l not in sa]
            inter.append(out)
            live[nxt] = out
            nxt += 1
        widths = [_log2size([dims_of[l] for l in t]) for t in inter]
        wmax = max(widths, default=0.0)
        if wmax <= max_log2:
            return sliced
        cand = {}
        for t, w in zip(inter, widths):
            if w >= wmax - 1e-9:
                for l in t:
                    if count.get(l) == 2 and l not in sliced:
                        cand[l] = cand.get(l, 0) + 1
        if not cand:
            return sliced
        cl = sorted(cand, key=lambda l: (-cand[l], l))[:candidates]
        best = None
        for l in cl:
            if time_model:
                f, w = path_model_cost(spec, path, sliced + [l]), 0.0
            else:
                f, w = _sliced_cost(spec, path, sliced + [l])
            key = (f, w, l)
            if best is None or key < best[0]:
                best = (key, l)
        sliced.append(best[1])


def slice_and_reconfigure(spec: NetworkSpec, path, max_log2: float, k: int = 10, rounds: int = 3,
                          time_model: bool = False):
    """Alternate exact slicing and subtree reconfiguration of the sliced network
    (cotengra's slice-and-reconfigure).  Returns (path, sliced, total flops,
    per-slice log2 width)."""
    sliced = []
    for _ in range(rounds):
        sliced = find_slices_exact(spec, path, max_log2, time_model=time_model)
        sub = _drop_labels(spec, sliced)
        path, _, _ = reconfigure_path(sub, path, k=k, passes=3, time_model=time_model)
    sliced = find_slices_exact(spec, path, max_log2, time_model=time_model)
    f, w = _sliced_cost(spec, path, sliced)
    return path, sliced, f, w


def hyper_path(spec: NetworkSpec, max_log2: float = 28.0, trials: int = 2, seed: int = 0,
               leaf: int = 14, k: int = 12, log=None, time_model: bool = False):
    """Sliced contraction plan for large circuits:
    presimplify (absorb rank <= 2 tensors) -> divisive partition tree
    (`partition_path`) -> subtree reconfiguration -> exact slicing alternated
    with reconfiguration until every per-slice intermediate is <= 2^max_log2.
    Best of `trials` seeds by total flops over all slices.  Returns
    (path over `spec`, sliced labels, total flops, per-slice log2 width)."""
    pre, ids, red = presimplify(spec)
    best = None
    for t in range(trials):
        s = seed + 1000 * t
        p, f, w = partition_path(red, trials=8, leaf=leaf, max_width=60, imbalance=(0.2, 0.8), seed=s)
        p, f, w = reconfigure_path(red, p, k=k, passes=3, seed=s)  # MAC model before slicing (measured better)
        p, sliced, fs, ws = slice_and_reconfigure(red, p, max_log2, k=k, rounds=2, time_model=time_model)
        score = path_model_cost(red, p, sliced, True) if time_model else fs
        if log:
            log(f"trial {t}: unsliced 2^{w:.0f} {f:.3g} flops -> {len(sliced)} sliced, 2^{ws:.0f}, "
                f"{fs:.3g} flops, model time {path_model_cost(red, p, sliced, True):.3g}")
        if best is None or score < best[4]:
            best = (p, sliced, fs, ws, score)
    p, sliced, fs, ws, _ = best
    return remap_path(pre, ids, len(spec.labels), p), sliced, fs, ws


def model_step_cost(wa: float, wb: float, wo: float, time_model: bool = True,
                    latency_macs: float = 1e4) -> float:
    """Cost of one pairwise step from the log2 sizes of its operands and result
    (FP32-tier MAC units).  MACs = 2^((wa+wb+wo)/2); with `time_model` the
    tensor-core tiers of dispatch_cgemm (precsel.cpp:275-306) are ~8x (TF32TCEC,
    min(m,n,k) >= 512) / ~14x (AUTO, >= 2048) faster than the bit-exact SIMT
    tier and every step pays an HBM floor of 8 B per operand/result element;
    few-output long-k steps pay the FP32 chain latency (~1e4 MACs per add)."""
    wk = (wa + wb - wo) / 2.0
    c = 2.0 ** ((wa + wb + wo) / 2.0)
    if time_model:
        wmin = min(wa - wk, wb - wk, wk)
        if wmin >= 11:
            c /= 14.0
        elif wmin >= 9:
            c /= 8.0
        c = max(c, 4.0 * (2.0 ** wa + 2.0 ** wb + 2.0 ** wo))
    if latency_macs and wo < 16.0:
        c += latency_macs * 2.0 ** wk
    return c


def path_model_cost(spec: NetworkSpec, path, drop=(), time_model: bool = True) -> float:
    """Sum of model_step_cost over the path with `drop` sliced, times the
    number of slices."""
    sub = _drop_labels(spec, drop)
    dims_of = {l: d for ls, ds in zip(spec.labels, spec.dims) for l, d in zip(ls, ds)}
    live = {i: list(ls) for i, ls in enumerate(sub.labels)}
    nxt = len(sub.labels)
    total = 0.0
    for a, b in path:
        la, lb = live.pop(a), live.pop(b)
        sa, sb = set(la), set(lb)
        out = [l for l in la if l not in sb] + [l for l in lb if l not in sa]
        total += model_step_cost(_log2size([dims_of[l] for l in la]), _log2size([dims_of[l] for l in lb]),
                                 _log2size([dims_of[l] for l in out]), time_model)
        live[nxt] = out
        nxt += 1
    return total * float(np.prod([dims_of[l] for l in drop])) if drop else total
