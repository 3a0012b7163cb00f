"""The canonical sum of the decomposed lattice (csrc/dd.cu): a balanced binary
tree over the values in index order, zero padded to a power of two.  The
kernels that produce row partials use different chunk widths — 4 columns in
the warp-marching stencil pass (csrc/march.cuh), 8-64 in the halo-tile and
update passes — and k_dd_rowred combines them chunk by chunk (coalesced
64-value chunks for long rows); strips hold power-of-two blocks of rows.
All of that only re-associates the SAME tree, so every global sum is the same
bits for every chunk width and strip count.  This pins that arithmetic fact
on the CPU (the GPU tests check the kernels against it indirectly)."""

import numpy as np


def tree(v):
    """Balanced tree in index order, zero padded to a power of two."""
    v = np.asarray(v, dtype=np.float64)
    n = 1
    while n < v.size:
        n *= 2
    a = np.zeros(n)
    a[:v.size] = v
    while a.size > 1:
        a = a[0::2] + a[1::2]
    return a[0]


def chunked(v, width):
    """Partials of `width` consecutive values, then the tree over the partials."""
    v = np.asarray(v, dtype=np.float64)
    pad = (-v.size) % width
    v = np.concatenate([v, np.zeros(pad)])
    return tree([tree(c) for c in v.reshape(-1, width)])


def test_row_sum_is_the_same_tree_for_every_power_of_two_chunk_width():
    rng = np.random.default_rng(0)
    for T in (8, 56, 96, 200, 2048):
        row = rng.standard_normal(T) * 10.0 ** rng.integers(-6, 6, T)
        want = tree(row)
        for w in (1, 2, 4, 8, 16, 32, 64):
            if T % w == 0:
                assert chunked(row, w) == want, (T, w)
        # the marching pass: 4-column partials of 28-column bands (a band is seven
        # whole groups), combined as k_dd_rowred does for long rows — 64-partial
        # chunks, then the chunk values
        parts = [tree(row[i:i + 4]) for i in range(0, T, 4)]
        assert chunked(parts, 64) == want, T


def test_lattice_sum_is_the_same_tree_for_every_strip_count():
    rng = np.random.default_rng(1)
    L, T = 64, 24
    site = rng.standard_normal((L, T))
    rows = [tree(r) for r in site]
    want = tree(rows)
    for G in (1, 2, 4, 8, 16, 32, 64):   # power-of-two strip heights are subtrees
        Lloc = L // G
        strips = [tree(rows[g * Lloc:(g + 1) * Lloc]) for g in range(G)]
        assert tree(strips) == want, G
    # a non-power-of-two strip height is NOT a subtree: the value may differ in
    # the last bits (why dd.py asks for power-of-two strip heights when
    # bit-identity across strip counts is wanted)
    odd = tree([tree(rows[g * 21:(g + 1) * 21]) for g in range(4)][:3] + [tree(rows[63:])])
    assert abs(odd - want) <= 1e-12 * max(1.0, abs(want))
