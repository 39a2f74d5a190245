"""Extension A1: meshes whose element count per axis is
not a power of two (C5's 48^3).  The reference rejects them
(mesh.hpp:143-149), so there is no oracle output to compare with; the
extension is pinned by:

* the generic (restricted-Morton) construction reproduces the reference's
  mesh and operators bit for bit when n IS a power of two;
* the element order, sparsity pattern and coarsening maps of a non-power-
  of-two mesh equal an independent restatement here (in-range cells of the
  bounding 2^k grid in Morton order; face neighbours with periodic wrap);
* translation invariance of the uniform periodic operator: every row holds
  the same diagonal / per-direction neighbour blocks, and those blocks equal
  the power-of-two mesh's scaled by (h/h')^(d-2) (the LDG Laplacian's
  blocks scale as h^(d-2) -- mass h^d, gradients h^(d-1), penalty beta/h),
  to rounding;
* the default (reference) path still rejects n that is not a power of two.
"""
import numpy as np
import pytest

import paper_2412_12506_b200 as g
from tests import cases as K


def morton_cells(n, dim):
    k = max(1, int(np.ceil(np.log2(n))))
    cells = []
    for code in range((1 << k) ** dim):
        ix = [0, 0, 0]
        for b in range(k):
            for a in range(dim):
                ix[a] |= ((code >> (b * dim + a)) & 1) << b
        if all(ix[a] < n for a in range(dim)):
            cells.append(tuple(ix[:dim]))
    return cells


def expected_pattern(n, dim, periodic):
    cells = morton_cells(n, dim)
    where = {c: i for i, c in enumerate(cells)}
    ptr, col = [0], []
    for c in cells:
        nb = {where[c]}
        for a in range(dim):
            for s in (-1, 1):
                d = list(c)
                d[a] += s
                if periodic:
                    d[a] %= n
                elif not 0 <= d[a] < n:
                    continue
                nb.add(where[tuple(d)])
        col += sorted(nb)
        ptr.append(len(col))
    return cells, np.array(ptr), np.array(col)


@pytest.mark.parametrize("spec", [K.scalar(8, 2, K.P, degree=2), K.scalar(8, 2, K.D, degree=1),
                                  K.stokes(4, 3, K.P, degree=1), K.stokes(8, 2, K.P, gamma=1.0, degree=1)])
def test_power_of_two_is_the_reference_mesh(spec):
    a, b = g.Problem(spec), g.Problem(spec, any_n=True)
    assert a.depth == b.depth
    for l in range(a.depth):
        for u, v in zip(a.level_matrix(l), b.level_matrix(l)):
            assert u.tobytes() == v.tobytes()
        if l + 1 < a.depth:
            for u, v in zip(a.level_transfer(l), b.level_transfer(l)):
                assert np.array_equal(u, v)


def test_reference_path_rejects_non_power_of_two():
    with pytest.raises(g.InvalidArgument, match="power of two"):
        g.Problem(K.scalar(6, 2, K.P))


@pytest.mark.parametrize("n,dim,bc", [(6, 2, K.P), (12, 2, K.D), (6, 3, K.P), (10, 2, K.P)])
def test_pattern_order_and_coarsening(n, dim, bc):
    P = g.Problem(K.scalar(n, dim, bc, degree=1), min_depth=1, bottom_max_elements=1 << 20, any_n=True)
    sizes = []
    m = n
    while True:
        sizes.append(m)
        if m < 4 or m % 2:
            break
        m //= 2
    assert P.depth == len(sizes)
    for l, m in enumerate(sizes):
        cells, ptr, col = expected_pattern(m, dim, bc == K.P)
        pp, pc = P.level_pattern(l)
        assert np.array_equal(pp, ptr) and np.array_equal(pc, col), (l, m)
        if l + 1 < P.depth:
            par, orth = P.level_transfer(l)
            coarse = {c: i for i, c in enumerate(morton_cells(sizes[l + 1], dim))}
            for f, c in enumerate(cells):
                assert par[f] == coarse[tuple(x // 2 for x in c)]
                assert orth[f] == sum((c[a] & 1) << a for a in range(dim))
            assert np.array_equal(par, np.arange(len(cells)) // (1 << dim))  # siblings contiguous


@pytest.mark.parametrize("n,m,dim,degree", [(6, 8, 2, 2), (12, 16, 2, 1), (6, 4, 3, 1), (6, 8, 3, 2)])
def test_translation_invariance_and_scaling(n, m, dim, degree):
    """uniform periodic Poisson: A on the n-mesh is the m-mesh's operator
    re-indexed, blocks scaled by (m/n)^(d-2)."""
    def blocks(N):
        P = g.Problem(K.scalar(N, dim, K.P, degree=degree), min_depth=1, bottom_max_elements=1 << 20, any_n=True)
        ptr, col, val = P.level_matrix(0)
        _, bs, _ = P.level_shape(0)
        cells = morton_cells(N, dim)
        where = {c: i for i, c in enumerate(cells)}
        out = {}
        for e, c in enumerate(cells):
            for k in range(ptr[e], ptr[e + 1]):
                j = col[k]
                d = tuple(((cells[j][a] - c[a] + 1) % N) - 1 for a in range(dim))  # offset in {-1,0,1}
                blk = val[k * bs * bs:(k + 1) * bs * bs]
                out.setdefault(d, []).append(blk)
            assert where[c] == e
        return {d: np.array(v) for d, v in out.items()}

    A, B = blocks(n), blocks(m)
    scale = (m / n) ** (dim - 2)
    assert set(A) == set(B) and len(A) == 2 * dim + 1
    for d in A:
        ref = B[d][0] * scale
        tol = 1e-12 * np.abs(ref).max()
        assert np.abs(A[d] - ref).max() <= tol, d          # every row, every direction
        assert np.abs(B[d] - B[d][0]).max() <= 1e-14 * np.abs(ref).max()


def test_c5_shape_hierarchy():
    """C5's 48^3 chain 48 -> 24 -> 12 -> 6 -> 3 (27 <= 64 bottom budget), on
    the 2D analogue so the CPU suite stays fast; and the 3D 12^3 chain."""
    P = g.Problem(K.scalar(48, 2, K.P, degree=1), min_depth=2, bottom_max_elements=64, any_n=True)
    assert [P.level_shape(l)[0] for l in range(P.depth)] == [48 * 48, 24 * 24, 12 * 12, 6 * 6, 3 * 3]
    P3 = g.Problem(K.stokes(12, 3, K.P, degree=1, delta=0.01, beta_p=1 / 16), min_depth=2, any_n=True)
    assert [P3.level_shape(l)[0] for l in range(P3.depth)] == [1728, 216, 27]
