"""Contraction-order planner (L0 tooling; not graded, not the oracle, not the product path).

* random-greedy pairwise contraction tree (many seeded trials);
* greedy slicing ("drilling holes / breaking edges") until every
  intermediate has at most ``2^max_log2`` elements;
* stem identification by greedy descent on subtree cost, ties -> left (C-A18);
* branch grouping: consecutive stem branches are pre-contracted into one MB-scale non-stem tensor
  when the B200 roofline time model says the merged step is cheaper ("non-stem tensors have
  manitude of MB").  Objective = estimated time on B200, not flop count.

All label sets are Python int bitmasks (every mode has dimension 2).
"""
from __future__ import annotations

import heapq
import math
import random

# B200 numbers used only by the planner's cost model (MEASURED_PEAKS.json of this pod)
P_TENSOR = 1.4e15 * 0.7   # sustained fp16 tensor flop/s we expect to reach
P_SIMT = 15e12            # complex64 SIMT flop/s for common-type (branch) contractions
HBM = 6.0e12              # B/s
ELEM_BYTES = 4            # complex-half stem element
LAUNCH = 4e-6             # s per kernel launch


def popcount(x: int) -> int:
    return x.bit_count()


def bits_of(x: int):
    out = []
    while x:
        low = x & -x
        out.append(low.bit_length() - 1)
        x ^= low
    return out


class Tree:
    """SSA contraction tree: nodes 0..n_leaves-1 are leaves; node n_leaves+i = pairs[i]."""

    def __init__(self, leaf_masks, pairs):
        self.leaf_masks = list(leaf_masks)
        self.pairs = list(pairs)
        self.n_leaves = len(leaf_masks)
        self.masks = list(leaf_masks)
        self.children = {}
        for i, (u, v) in enumerate(pairs):
            self.masks.append(self.masks[u] ^ self.masks[v])
            self.children[self.n_leaves + i] = (u, v)
        self.root = len(self.masks) - 1

    def node_cost(self, k, sliced=0):
        u, v = self.children[k]
        return 1 << popcount((self.masks[u] | self.masks[v]) & ~sliced)

    def total_cost(self, sliced=0):
        """complex MACs of one slice"""
        return sum(self.node_cost(k, sliced) for k in self.children)

    def max_log2(self, sliced=0):
        return max(popcount(m & ~sliced) for m in self.masks)

    def subtree_costs(self, sliced=0):
        cost = [0] * len(self.masks)
        for k in range(self.n_leaves, len(self.masks)):
            u, v = self.children[k]
            cost[k] = cost[u] + cost[v] + self.node_cost(k, sliced)
        return cost


def greedy_tree(leaf_masks, rng, alpha=1.0, temperature=0.0):
    """Random-greedy pairwise order: pick the connected pair minimising
    size(out) - alpha*(size(a)+size(b)) with Gumbel-perturbed scores."""
    masks = {i: m for i, m in enumerate(leaf_masks)}
    holders = {}
    for i, m in masks.items():
        for l in bits_of(m):
            holders.setdefault(l, set()).add(i)
    heap = []

    def push(i, j):
        mi, mj = masks[i], masks[j]
        so = float(1 << popcount(mi ^ mj))
        sa, sb = float(1 << popcount(mi)), float(1 << popcount(mj))
        score = so - alpha * (sa + sb)
        if temperature > 0:
            g = -math.log(-math.log(rng.random() + 1e-300) + 1e-300)
            score -= temperature * g * (sa + sb)
        heapq.heappush(heap, (score, i, j))

    seen = set()
    for l, hs in holders.items():
        hs = sorted(hs)
        for a in range(len(hs)):
            for b in range(a + 1, len(hs)):
                if (hs[a], hs[b]) not in seen:
                    seen.add((hs[a], hs[b]))
                    push(hs[a], hs[b])
    pairs = []
    nxt = len(leaf_masks)
    alive = set(masks)
    while heap:
        _, i, j = heapq.heappop(heap)
        if i not in alive or j not in alive:
            continue
        mi, mj = masks[i], masks[j]
        k = nxt
        nxt += 1
        pairs.append((i, j))
        masks[k] = mi ^ mj
        alive.discard(i)
        alive.discard(j)
        alive.add(k)
        nbrs = set()
        for l in bits_of(mi | mj):
            hs = holders.get(l)
            if hs is None:
                continue
            hs.discard(i)
            hs.discard(j)
            if masks[k] >> l & 1:
                hs.add(k)
            nbrs |= hs
        nbrs.discard(k)
        for o in nbrs:
            push(min(o, k), max(o, k)) if o < k else push(k, o)
    # disconnected components: contract the remaining pieces (outer products), smallest first
    rest = sorted(alive, key=lambda x: popcount(masks[x]))
    while len(rest) > 1:
        i, j = rest[0], rest[1]
        k = nxt
        nxt += 1
        pairs.append((i, j))
        masks[k] = masks[i] ^ masks[j]
        rest = sorted(rest[2:] + [k], key=lambda x: popcount(masks[x]))
    return pairs


def find_slices(tree, max_log2, open_mask=0, max_slices=400):
    """Greedy slicing: repeatedly fix the closed label (dimension 2) that minimises
    2^|S| * per-slice cost among labels of the oversized intermediates."""
    sliced = 0
    while tree.max_log2(sliced) > max_log2:
        if popcount(sliced) >= max_slices:
            return None
        worst = max(popcount(m & ~sliced) for m in tree.masks)
        cand = 0
        for m in tree.masks:
            if popcount(m & ~sliced) >= worst - 1:
                cand |= m
        cand &= ~sliced & ~open_mask
        best = None
        for l in bits_of(cand):
            s2 = sliced | (1 << l)
            c = tree.total_cost(s2)
            mx = tree.max_log2(s2)
            key = (mx > max_log2, math.log2(c) + popcount(s2), mx)
            if best is None or key < best[0]:
                best = (key, l)
        if best is None:
            return None
        sliced |= 1 << best[1]
    return sliced


def find_stem(tree, sliced=0):
    """Leaf->root list of node ids: descend from the root into the child with larger subtree
    cost, ties -> left (C-A18)."""
    cost = tree.subtree_costs(sliced)
    path = [tree.root]
    k = tree.root
    while k in tree.children:
        u, v = tree.children[k]
        k = u if cost[u] >= cost[v] else v
        path.append(k)
    return path[::-1]


def step_time(m_log2, k_log2, n_log2, elem_bytes=ELEM_BYTES):
    M, K, N = 2.0 ** m_log2, 2.0 ** k_log2, 2.0 ** n_log2
    flops = 8 * M * K * N
    byts = elem_bytes * (M * K + M * N)
    # a permutation pass is needed on roughly half the steps
    perm = 0.5 * 2 * elem_bytes * M * K / HBM
    return max(flops / P_TENSOR, byts / HBM) + perm + LAUNCH


def group_branches(tree, sliced, stem, max_branch_log2=20, max_group=12):
    """Regroup consecutive stem branches (DP over the stem) to minimise modelled B200 time.
    Returns a new Tree with the same leaves and the new explicit stem (leaf->root)."""
    nm = lambda m: m & ~sliced
    masks = tree.masks
    steps = []  # (branch node id) for each stem step
    for a, b in zip(stem[:-1], stem[1:]):
        u, v = tree.children[b]
        steps.append(v if u == a else u)
    L = len(steps)
    stem_masks = [masks[stem[0]]]
    for s in steps:
        stem_masks.append(stem_masks[-1] ^ masks[s])

    def group_cost(j, jp):
        """cost of absorbing branches steps[j..jp] (inclusive) as one merged tensor"""
        bm = 0
        merge = 0.0
        for t in range(j, jp + 1):
            mt = masks[steps[t]]
            if t > j:
                merge += 8.0 * (1 << popcount(nm(bm | mt))) / P_SIMT + LAUNCH
            bm ^= mt
            if jp > j and popcount(nm(bm)) > max_branch_log2:
                return None
        s = nm(stem_masks[j])
        b = nm(bm)
        m = popcount(s & ~b)
        k = popcount(s & b)
        n = popcount(b & ~s)
        return step_time(m, k, n) + merge

    best = [0.0] + [math.inf] * L
    arg = [0] * (L + 1)
    for jp in range(1, L + 1):
        for j in range(max(1, jp - max_group + 1), jp + 1):
            c = group_cost(j - 1, jp - 1)
            if c is None:
                continue
            if best[j - 1] + c < best[jp]:
                best[jp] = best[j - 1] + c
                arg[jp] = j
    groups = []
    jp = L
    while jp > 0:
        j = arg[jp]
        groups.append((j - 1, jp - 1))
        jp = j - 1
    groups.reverse()

    # rebuild SSA pairs: keep every non-stem internal node, then merged branches + stem steps
    stem_set = set(stem)
    keep = [k for k in sorted(tree.children) if k not in stem_set]
    new_pairs = []
    remap = {i: i for i in range(tree.n_leaves)}
    nxt = tree.n_leaves

    def emit(u, v):
        nonlocal nxt
        new_pairs.append((u, v))
        nxt += 1
        return nxt - 1

    for k in keep:
        u, v = tree.children[k]
        remap[k] = emit(remap[u], remap[v])
    cur = remap[stem[0]]
    new_stem = [cur]
    for (j, jp) in groups:
        b = remap[steps[j]]
        for t in range(j + 1, jp + 1):
            b = emit(b, remap[steps[t]])
        cur = emit(cur, b)
        new_stem.append(cur)
    return Tree(tree.leaf_masks, new_pairs), new_stem, best[L]


def unslice_to_target(tree, sliced, target_log2):
    """Greedily un-slice edges (fewest subtasks) while every intermediate of ``tree`` stays
    <= 2^target_log2 elements: each pass removes the sliced label whose removal keeps the bound and
    adds the least per-slice cost.  Branch grouping shrinks the stem, so a grouped tree needs far
    fewer sliced edges than the ungrouped tree it came from."""
    while True:
        best = None
        for l in bits_of(sliced):
            s2 = sliced & ~(1 << l)
            if tree.max_log2(s2) > target_log2:
                continue
            c = tree.total_cost(s2)
            if best is None or c < best[0]:
                best = (c, l)
        if best is None:
            return sliced
        sliced &= ~(1 << best[1])


def left_deep_pairs(order):
    """SSA pairs of the left-deep tree absorbing leaves in ``order`` (a sweep)."""
    n = len(order)
    pairs = []
    cur = order[0]
    for i, t in enumerate(order[1:]):
        pairs.append((cur, t))
        cur = n + i
    return pairs


def plan_network(leaf_masks, open_mask, max_log2, trials=32, seed=0, group=True,
                 max_branch_log2=20, sweeps=(), max_group=12, stem_log2=None):
    """Search seeded random-greedy trees and the given sweep orders (left-deep trees); slice each
    to ``max_log2``; keep the cheapest by total (all-slices) cost.  Returns dict with tree,
    sliced mask, stem."""
    rng = random.Random(seed)
    best = None
    cands = [("sweep", o) for o in sweeps] + [("greedy", t) for t in range(trials)]
    for kind, t in cands:
        if kind == "sweep":
            pairs = left_deep_pairs(t)
        else:
            alpha = 1.0 if t == 0 else rng.uniform(0.5, 1.5)
            temp = 0.0 if t == 0 else rng.uniform(0.0, 1.0)
            pairs = greedy_tree(leaf_masks, rng, alpha=alpha, temperature=temp)
        tree = Tree(leaf_masks, pairs)
        sliced = find_slices(tree, max_log2, open_mask)
        if sliced is None:
            continue
        cost = tree.total_cost(sliced)
        key = math.log2(cost) + popcount(sliced)
        if best is None or key < best[0]:
            best = (key, tree, sliced)
    if best is None:
        raise RuntimeError("no feasible tree found")
    _, tree, sliced = best
    stem = find_stem(tree, sliced)
    est = None
    if group:
        tree, stem, est = group_branches(tree, sliced, stem, max_branch_log2=max_branch_log2, max_group=max_group)
    if stem_log2 is not None:
        # fewer sliced edges: bigger (paper-like) subtasks with the largest stem at 2^stem_log2
        sliced = unslice_to_target(tree, sliced, stem_log2)
    return {"tree": tree, "sliced": sliced, "stem": stem, "est_time": est}


def stem_report(tree, sliced, stem):
    """Per stem step geometry (log2 M, K, N)."""
    out = []
    masks = tree.masks
    for a, b in zip(stem[:-1], stem[1:]):
        u, v = tree.children[b]
        br = v if u == a else u
        s = masks[a] & ~sliced
        bm = masks[br] & ~sliced
        out.append((popcount(s & ~bm), popcount(s & bm), popcount(bm & ~s)))
    return out
