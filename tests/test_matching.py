"""Matching: reference Suitor vs restatement vs greedy vs the GPU parallel Suitor.

CPU: the restatement (mode 0) equals the compiled reference suitor_match on
random graphs with heavy ties; the total-order rule (mode 1) equals the greedy
matching under key(e) = (w, -min, -max); both are >= 1/2 of the brute-force
maximum weight matching (acceptance criterion 6).
GPU: the 128-bit-CAS parallel Suitor equals mode 1 exactly.
"""
import itertools
import os

import numpy as np
import pytest

import oracle

REF_OK = os.path.exists(oracle.LIBS["reference"])


def random_graph(n, p_edge, rng, levels=None):
    """Symmetric weighted graph CSR; weights from a small set when `levels` (ties)."""
    edges = {}
    for i in range(n):
        for j in range(i + 1, n):
            if rng.random() < p_edge:
                w = float(rng.integers(0, levels)) / levels if levels else float(rng.standard_normal())
                edges[(i, j)] = w
    adj = [[] for _ in range(n)]
    for (i, j), w in edges.items():
        adj[i].append((j, w))
        adj[j].append((i, w))
    rp, col, wt = [0], [], []
    for i in range(n):
        for j, w in sorted(adj[i]):
            col.append(j)
            wt.append(w)
        rp.append(len(col))
    return np.array(rp, np.int64), np.array(col, np.int64), np.array(wt), edges


def greedy(n, edges):
    order = sorted(edges.items(), key=lambda e: (-e[1], e[0][0], e[0][1]))
    mate = [-1] * n
    for (i, j), _ in order:
        if mate[i] == -1 and mate[j] == -1:
            mate[i], mate[j] = j, i
    return np.array(mate)


def weight_of(mate, edges):
    return sum(edges[(i, int(j))] for i, j in enumerate(mate) if j > i)


def brute_max(n, edges):
    best = 0.0
    items = list(edges.items())

    def rec(k, used, acc):
        nonlocal best
        best = max(best, acc)
        for t in range(k, len(items)):
            (i, j), w = items[t]
            if w > 0 and i not in used and j not in used:
                rec(t + 1, used | {i, j}, acc + w)

    rec(0, frozenset(), 0.0)
    return best


@pytest.mark.skipif(not REF_OK, reason="oracle/_ref not built")
@pytest.mark.parametrize("seed", range(40))
def test_restatement_equals_reference_suitor(seed):
    rng = np.random.default_rng(seed)
    rp, col, w, _ = random_graph(int(rng.integers(2, 40)), 0.2, rng, levels=int(rng.integers(1, 4)) or None)
    np.testing.assert_array_equal(oracle.match_graph("reference", rp, col, w), oracle.match_graph("restatement", rp, col, w, 0))


@pytest.mark.parametrize("seed", range(60))
def test_total_order_equals_greedy(seed):
    rng = np.random.default_rng(1000 + seed)
    n = int(rng.integers(2, 50))
    rp, col, w, edges = random_graph(n, 0.15, rng, levels=[None, 1, 2, 3][seed % 4])
    np.testing.assert_array_equal(oracle.match_graph("restatement", rp, col, w, 1), greedy(n, edges))


@pytest.mark.parametrize("seed", range(50))
def test_half_approximation(seed):
    rng = np.random.default_rng(2000 + seed)
    n = int(rng.integers(2, 12))
    rp, col, w, edges = random_graph(n, 0.4, rng)
    edges = {k: abs(v) for k, v in edges.items()}
    w = np.abs(w)
    opt = brute_max(n, edges)
    for mode in (0, 1):
        m = oracle.match_graph("restatement", rp, col, w, mode)
        assert weight_of(m, edges) >= 0.5 * opt - 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(30))
def test_gpu_suitor_equals_total_order(seed):
    import paper_2303_02352_b200 as pb

    rt = pb.Runtime(0, 0, 1)
    rng = np.random.default_rng(3000 + seed)
    n = int(rng.integers(2, 4000))
    rp, col, w, edges = random_graph(min(n, 300), 0.05, rng, levels=[None, 1, 2, 5][seed % 4])
    np.testing.assert_array_equal(pb.match_graph(rt, rp, col, w), oracle.match_graph("restatement", rp, col, w, 1))


@pytest.mark.gpu
@pytest.mark.parametrize("nd", [8, 17, 32])
def test_gpu_suitor_poisson_ties(nd):
    """All fine-level Poisson weights tie (7/6): worst case for contention."""
    import paper_2303_02352_b200 as pb

    rt = pb.Runtime(0, 0, 1)
    rp, ci, va = pb.poisson(7, nd, nd, nd)
    grp, gcol, gw = oracle.build_weights("restatement", rp, ci, va, np.ones(nd ** 3))
    np.testing.assert_array_equal(pb.match_graph(rt, grp, gcol, gw), oracle.match_graph("restatement", grp, gcol, gw, 1))
