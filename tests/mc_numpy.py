"""Marching cubes restated in numpy with the product's generated triangulation (api.mc_case):
test infrastructure for the GPU kernel (tests/test_gpu_mc.py compares it exactly) and for the
geometric comparison with the reference's own marching_cubes (mesh.hpp:75-156).

Conventions of mesh.hpp:36-46 (Bourke corners, an edge keyed by its lower node and axis),
vertex = a + t (b - a) with t = clamp((iso - v0) / (v1 - v0), 0, 1) (0.5 for a zero denominator),
welding of identical positions, triangles with a repeated vertex or area < 1e-12 dropped,
vertices numbered by first use."""
import numpy as np

CORNER = [(0, 0, 0), (1, 0, 0), (1, 1, 0), (0, 1, 0), (0, 0, 1), (1, 0, 1), (1, 1, 1), (0, 1, 1)]
EDGE_BASE = [0, 1, 3, 0, 4, 5, 7, 4, 0, 1, 2, 3]
EDGE_AXIS = [0, 1, 0, 1, 0, 1, 0, 1, 2, 2, 2, 2]


def node_pos(i, j, k, cells):
    r = float(cells)
    return (-1.0 + 2.0 * i / r, -1.0 + 2.0 * j / r, 1.0 - 2.0 * k / r)


def marching_cubes(values, cells, table, iso=0.5):
    n = cells + 1
    v = np.asarray(values, np.float32).reshape(n, n, n)  # [k, j, i]
    keyed = {}
    tris = []

    def vkey(i, j, k, ax):
        i1, j1, k1 = i + (ax == 0), j + (ax == 1), k + (ax == 2)
        v0, v1 = float(v[k, j, i]), float(v[k1, j1, i1])
        den = v1 - v0
        t = 0.5 if abs(den) < 1e-300 else (iso - v0) / den
        t = min(max(t, 0.0), 1.0)
        if t == 0.0:
            return ("n", i, j, k), node_pos(i, j, k, cells)
        if t == 1.0:
            return ("n", i1, j1, k1), node_pos(i1, j1, k1, cells)
        a, b = node_pos(i, j, k, cells), node_pos(i1, j1, k1, cells)
        return ("e", i, j, k, ax), tuple(a[d] + t * (b[d] - a[d]) for d in range(3))

    inside = v < iso
    for k in range(cells):
        for j in range(cells):
            for i in range(cells):
                cs = 0
                for c, (oi, oj, ok) in enumerate(CORNER):
                    if inside[k + ok, j + oj, i + oi]:
                        cs |= 1 << c
                for tri in table[cs]:
                    ids = []
                    for e in tri:
                        oi, oj, ok = CORNER[EDGE_BASE[e]]
                        key, pos = vkey(i + oi, j + oj, k + ok, EDGE_AXIS[e])
                        keyed.setdefault(key, pos)
                        ids.append(key)
                    tris.append(ids)
    out_v, out_t, used = [], [], {}
    for ids in tris:
        if ids[0] == ids[1] or ids[1] == ids[2] or ids[0] == ids[2]:
            continue
        p = [np.array(keyed[x]) for x in ids]
        if 0.5 * np.linalg.norm(np.cross(p[1] - p[0], p[2] - p[0])) < 1e-12:
            continue
        r = []
        for x in ids:
            if x not in used:
                used[x] = len(out_v)
                out_v.append(keyed[x])
            r.append(used[x])
        out_t.append(r)
    return np.array(out_v, np.float64).reshape(-1, 3), np.array(out_t, np.int32).reshape(-1, 3)


def edge_use_counts(tris):
    """Undirected edge -> number of triangles using it (2 everywhere for a closed manifold)."""
    cnt = {}
    for a, b, c in tris:
        for x, y in ((a, b), (b, c), (c, a)):
            e = (min(x, y), max(x, y))
            cnt[e] = cnt.get(e, 0) + 1
    return cnt


def area_and_volume(verts, tris):
    p = verts[tris]
    cr = np.cross(p[:, 1] - p[:, 0], p[:, 2] - p[:, 0])
    area = 0.5 * np.linalg.norm(cr, axis=1).sum()
    vol = np.einsum("ij,ij->i", p[:, 0], np.cross(p[:, 1], p[:, 2])).sum() / 6.0
    return area, vol
