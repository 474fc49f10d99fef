"""CPU checks of the seeded input generators (workloads/), which hold no method arithmetic."""
import numpy as np

from workloads import c2_lattice, c2_grids, MICROBENCH
from oracle.tree import Level, interaction_list


class _Periodic(dict):
    def __init__(self, g, dims):
        super().__init__()
        self.dims = dims
        self.pos = {tuple(int(v) for v in c): k for k, c in enumerate(g)}

    def get(self, c, default=None):
        return self.pos.get(tuple(int(c[d]) % self.dims[d] for d in range(3)), default)


def test_c2_lattice_is_the_oracle_interaction_list():
    """C2 microbench CSR == oracle.tree.interaction_list on the periodic lattice; 189 each."""
    g, row, src, oid, offs = c2_lattice()
    assert len(g) == MICROBENCH["boxes"] == 64 * 32 * 32
    assert len(offs) == 316 and np.all(np.diff(row) == 189)
    assert len({tuple(c) for c in g}) == len(g)
    lev = Level(0, 1.0, [tuple(c) for c in g], _Periodic(g, MICROBENCH["lattice"]), [], np.zeros((len(g), 3)))
    tid = {tuple(int(v) for v in o): k for k, o in enumerate(offs)}
    rng = np.random.default_rng(0)
    for a in np.concatenate([[0, len(g) - 1], rng.choice(len(g), 30, replace=False)]):
        il = interaction_list(lev, tuple(int(v) for v in g[a]))
        assert sorted((int(k), tid[o]) for k, o in il) == sorted(zip(src[row[a]:row[a + 1]].tolist(),
                                                                     oid[row[a]:row[a + 1]].tolist()))


def test_c2_morton_order_locality():
    """Boxes are in Morton order: each aligned 2x2x2 sibling group is 8 consecutive boxes."""
    g, *_ = c2_lattice()
    par = g >> 1
    assert np.all(par[0::8][:, None, :] == par.reshape(-1, 8, 3))
    assert c2_grids(8) == ((16, 16), (32, 32))
