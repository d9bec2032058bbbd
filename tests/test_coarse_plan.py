"""Host logic of the nested-dissection coarse solve (coarse.cu nd_plan, exported as
cr_coarse_nd_plan), checked on CPU against the conditions that make the
multifrontal elimination exact, recomputed here by brute force:
  * every coarse node is a pivot of exactly one front; children precede parents (post-order);
  * separation: two nodes coupled by the 5^d-node stencil of Z^t G Z are pivots of fronts on
    one root path (otherwise eliminating one would fill in between independent subtrees);
  * each front's B set is exactly the set of later-eliminated nodes coupled to its subtree,
    ordered by (front, node)."""
import itertools

import numpy as np
import pytest

import paper_2101_03777_b200 as P


def _coords(v, H, d):
    c = []
    for _ in range(d):
        c.append(v % (H + 1))
        v //= H + 1
    return np.array(c)


@pytest.mark.parametrize("H,d,box", [(1, 2, 0), (3, 2, 0), (8, 2, 0), (13, 2, 0), (21, 2, 0), (2, 3, 0), (5, 3, 0),
                                     (8, 3, 0), (21, 2, 4), (24, 2, 6), (11, 2, 8), (9, 3, 3), (2, 2, 4)])
def test_nd_plan_is_a_valid_elimination(H, d, box):
    pl = P.coarse_nd_plan(H, d, box)
    nf = len(pl["I"])
    nn = (H + 1) ** d
    pos = np.full(nn, -1)
    for f in range(nf):
        for v in pl["I"][f]:
            assert pos[v] == -1, "node in two fronts"
            pos[v] = f
    assert (pos >= 0).all()
    parent = pl["parent"].astype(int)
    for f in range(nf):
        if parent[f] >= 0:
            assert f < parent[f]
            assert pl["depth"][f] == pl["depth"][parent[f]] + 1
    assert (parent == -1).sum() == 1 and parent[nf - 1] == -1
    anc = [set() for _ in range(nf)]
    for f in range(nf):
        g = f
        while g >= 0:
            anc[f].add(g)
            g = parent[g]
    sub = [set() for _ in range(nf)]
    for f in range(nf):
        for g in anc[f]:
            sub[g].add(f)
    offs = [np.array(o) for o in itertools.product(range(-2, 3), repeat=d)]
    coupled = [[] for _ in range(nn)]
    for v in range(nn):
        cv = _coords(v, H, d)
        for o in offs:
            w = cv + o
            if (w >= 0).all() and (w <= H).all():
                coupled[v].append(int(sum(int(w[i]) * (H + 1) ** i for i in range(d))))
    for v in range(nn):
        for u in coupled[v]:
            fu, fv = pos[u], pos[v]
            assert fu in anc[fv] or fv in anc[fu], (u, v, fu, fv)
    for f in range(nf):
        nodes = [v for g in sub[f] for v in pl["I"][g]]
        expect = {u for v in nodes for u in coupled[v] if pos[u] not in sub[f]}
        assert set(pl["B"][f].tolist()) == expect, f
        key = [(pos[u], u) for u in pl["B"][f]]
        assert key == sorted(key)
        assert all(pos[u] in anc[f] for u in pl["B"][f])
