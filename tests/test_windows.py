"""Node-window arrays (device.window_arrays, the layout registered through
ab_set_windows / ab_set_window_refs) built on the CPU: every element-node
reference resolves to its node through the window, and the slot lists and
the sorted reference records cover every reference exactly once."""

import numpy as np
import pytest
import torch

from paper_2005_05899_b200 import meshgen
from paper_2005_05899_b200.device import WINDOW_BLOCK, window_arrays


def _conn(name):
    if name == "tet":
        m = meshgen.box_tets(9, 8, 7, jitter=0.2, seed=4)
        c = m.conn["tet4"]
    else:
        m = meshgen.box_hexes(7, 6, 9)
        c = m.conn["hex8"]
    # a shuffled element order exercises arbitrary windows; the SFC order is a special case
    rng = np.random.default_rng(1)
    c = c[rng.permutation(len(c))][: len(c) - 37]  # ragged last block
    return torch.from_numpy(np.ascontiguousarray(c, dtype=np.int32)), m.n_nodes


@pytest.mark.parametrize("name", ["tet", "hex"])
def test_window_arrays_consistent(name):
    conn, N = _conn(name)
    E, nn = conn.shape
    B = WINDOW_BLOCK
    blk_ptr, wnode, wptr, wslot, loc, wmax, desc, wref = window_arrays(conn, N, B)
    c = conn.numpy().astype(np.int64)
    bp = blk_ptr.numpy()
    wn = wnode.numpy()[: bp[-1]].astype(np.int64)
    lc = loc.numpy()[:E].reshape(E, nn).astype(np.int64)
    nblk = (E + B - 1) // B
    assert len(bp) == nblk + 1 and (np.diff(bp) <= wmax).all()
    # element side: window index -> node
    blk = np.arange(E) // B
    assert np.array_equal(wn[bp[blk][:, None] + lc], c)
    # owner side: every slot offset a*B + e%B appears exactly once, in its node's list
    wp = wptr.numpy().astype(np.int64)
    ws = wslot.numpy().astype(np.int64) & 0xFFFF
    seen = np.zeros((nblk, nn * B), dtype=np.int64)
    for b in range(nblk):
        for k in range(bp[b], bp[b + 1]):
            for t in range(wp[k], wp[k + 1]):
                off = ws[t]
                e = b * B + off % B
                a = off // B
                assert e < E and c[e, a] == wn[k]
                seen[b, off] += 1
    valid = (np.arange(nblk)[:, None] * B + np.arange(nn * B)[None, :] % B) < E
    assert (seen[valid] == 1).all() and (seen[~valid] == 0).all()
    # sorted references: runs of equal window index, each reference once, padding 0xffff
    wr = wref.numpy().astype(np.int64) & 0xFFFFFFFF
    assert len(wr) == nblk * B * nn
    for b in range(nblk):
        rec = wr[b * B * nn:(b + 1) * B * nn]
        li, off = rec >> 16, rec & 0xFFFF
        real = li != 0xFFFF
        assert np.all(np.diff(li[real]) >= 0)  # sorted by window index
        e = b * B + off[real] % B
        assert np.array_equal(wn[bp[b] + li[real]], c[e, off[real] // B])
        assert len(np.unique(off[real])) == real.sum() == min(B, E - b * B) * nn
    # descriptors
    d = desc.numpy().astype(np.int64)
    assert np.array_equal(d[:, 0], bp[:-1]) and np.array_equal(d[:, 1], bp[1:])
    assert np.array_equal(d[:, 2], wp[bp[:-1]]) and np.array_equal(d[:, 3], wp[bp[1:]])
