"""Pins of oracle.nearlist (row a2)."""
import numpy as np
from scipy.spatial import cKDTree

import nat_inputs as I
from oracle import geometry, nearlist


def test_class_S_counts_from_vertex_valence():
    m = I.icosphere(2)
    g = geometry.mesh_prepare(m.v, m.t)
    rp, col, cls = nearlist.near_list(m.t, g["centroid"], g["diam"])
    val = np.bincount(m.t.ravel(), minlength=m.n_vert)
    for i in range(m.n_tri):
        # triangles around the 3 vertices, minus T_i itself counted 3x, minus the 3
        # edge neighbours counted twice
        expect = int(val[m.t[i]].sum()) - 3 - 3
        assert int(np.sum(cls[rp[i]:rp[i + 1]] == nearlist.CLS_S)) == expect


def test_class_N_matches_kdtree_and_csr_sorted():
    m = I.bowl(32, 8, 2)
    g = geometry.mesh_prepare(m.v, m.t)
    eta = 4.0
    rp, col, cls = nearlist.near_list(m.t, g["centroid"], g["diam"], eta)
    tree = cKDTree(g["centroid"])
    near = [set() for _ in range(m.n_tri)]
    for j in range(m.n_tri):                      # i within eta*diam_j of c_j
        for i in tree.query_ball_point(g["centroid"][j], eta * g["diam"][j] * (1 - 1e-12)):
            if i != j:
                near[i].add(j)
    vs = [set(map(int, tri)) for tri in m.t]
    for i in range(m.n_tri):
        cols = col[rp[i]:rp[i + 1]]
        assert np.all(np.diff(cols) > 0)
        S = {int(j) for j, c in zip(cols, cls[rp[i]:rp[i + 1]]) if c == nearlist.CLS_S}
        N = {int(j) for j, c in zip(cols, cls[rp[i]:rp[i + 1]]) if c == nearlist.CLS_N}
        assert S == {j for j in range(m.n_tri) if j != i and vs[i] & vs[j]}
        assert N == near[i] - S
