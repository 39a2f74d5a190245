"""Ghost-layer size of the C5 48^3 partition choices.

Contiguous ranges of the restricted Morton order (extension A1, the order the
partitioned V-cycle uses: partition_ranges, smoothers.hpp:87-94) against
z-slabs of 48/P layers, on the periodic face-neighbour graph (the gamma = 0
operator's stencil away from the interface).  Prints, per P, the largest and
total ghost element counts (one ghost element = one 108-double block in the
exchange) and whether each choice is nested across the levels 48 -> 24 -> 12
(so that restriction / prolongation stay rank-local).

  python tools/ghost_analysis.py [n]
"""
import json
import sys

import numpy as np


def morton_cells(n, dim=3):
    """Cells of the n^dim grid in the Morton order of the bounding 2^k grid."""
    k = max(1, int(np.ceil(np.log2(n))))
    idx = np.arange(n)
    g = np.stack(np.meshgrid(*([idx] * dim), indexing="ij"), -1).reshape(-1, dim)
    code = np.zeros(len(g), np.int64)
    for b in range(k):
        for a in range(dim):
            code |= ((g[:, a] >> b) & 1).astype(np.int64) << (b * dim + a)
    return g[np.argsort(code, kind="stable")]


def ghosts(owner, cells, n, P):
    pos = {tuple(c): i for i, c in enumerate(cells)}
    nb_owner = []
    for a in range(3):
        for s in (-1, 1):
            sh = cells.copy()
            sh[:, a] = (sh[:, a] + s) % n
            nb_owner.append(np.array([owner[pos[tuple(c)]] for c in sh]))
    nb_owner = np.stack(nb_owner, 1)
    per = []
    for p in range(P):
        rows = owner == p
        ids = set()
        for a in range(6):
            m = rows & (nb_owner[:, a] != p)
            sh = cells[m].copy()
            ax, s = a // 2, (-1, 1)[a % 2]
            sh[:, ax] = (sh[:, ax] + s) % n
            ids.update(map(tuple, sh))
        per.append(len(ids))
    return per


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 48
    cells = morton_cells(n)
    N = len(cells)
    out = {}
    for P in (2, 4, 8):
        morton = np.empty(N, int)
        for p in range(P):
            morton[p * N // P:(p + 1) * N // P] = p
        slab = cells[:, 2] * P // n
        gm, gs = ghosts(morton, cells, n, P), ghosts(slab, cells, n, P)
        # nesting: a coarse cell's 8 children must share an owner (levels 48 -> 24 -> 12)
        def nested(owner, cells_f):
            par = {}
            for o, c in zip(owner, cells_f):
                par.setdefault(tuple(c // 2), set()).add(int(o))
            return all(len(v) == 1 for v in par.values())
        out[P] = {"morton_ghosts_max": max(gm), "morton_ghosts_total": sum(gm),
                  "slab_ghosts_max": max(gs), "slab_ghosts_total": sum(gs),
                  "morton_nested": nested(morton, cells), "slab_nested": nested(slab, cells),
                  "exchange_MB_per_neighbour_layer_morton_max": max(gm) * 108 * 8 / 1e6}
        print(P, json.dumps(out[P]), flush=True)


if __name__ == "__main__":
    main()
