"""The symmetric-orbit decomposition of the diagonal layer blocks (DESIGN.md
section 2, csrc/symkr.cuh, Engine::orbit_block) checked on the CPU:

* every entry of a diagonal block (weights and biases, index T_k = the bias)
  is one of the four images of exactly one representative (i <= c, o <= o''),
* the reference's own H and G (golden fixtures from oracle/_ref) are constant
  on every orbit, for every layer of every smooth golden case,
* the orbit-tile shard ranges the kernels use for row shards partition the
  representatives.
"""
import numpy as np
import pytest

from conftest import load_golden


def block_index(widths, k):
    """Canonical flat index of (unit o, input x) of step k; x = T_k is the bias."""
    off = 0
    for s in range(k):
        off += widths[s + 1] * (widths[s] + 1)
    tk, u = widths[k], widths[k + 1]
    return lambda o, x: off + o * tk + x if x < tk else off + u * tk + o


def orbit_images(o, i, oo, c):
    return {(o, i, oo, c), (oo, c, o, i), (o, c, oo, i), (oo, i, o, c)}


@pytest.mark.parametrize("tk,u", [(4, 3), (3, 5), (1, 1), (6, 2)])
def test_orbits_cover_each_entry_once(tk, u):
    seen = {}
    for i in range(tk + 1):
        for c in range(i, tk + 1):
            for o in range(u):
                for oo in range(o, u):
                    for e in orbit_images(o, i, oo, c):
                        seen.setdefault(e, set()).add((o, i, oo, c))
    # every (unit, input) x (unit, input) pair of the block, exactly one representative
    assert len(seen) == (u * (tk + 1)) ** 2
    assert all(len(reps) == 1 for reps in seen.values())


@pytest.mark.parametrize("name", ["config0", "tanh352", "sigmoid654", "deep4653", "logistic32"])
def test_reference_curvature_is_constant_on_orbits(name):
    g = load_golden(name)
    widths = g["spec"]["widths"]
    for mat in ("H", "G"):
        M = g[mat]
        scale = max(1.0, np.abs(M).max())
        for k in range(len(widths) - 1):
            tk, u = widths[k], widths[k + 1]
            idx = block_index(widths, k)
            for i in range(tk + 1):
                for c in range(i, tk + 1):
                    for o in range(u):
                        for oo in range(o, u):
                            vals = [M[idx(a, x), idx(b, y)] for a, x, b, y in orbit_images(o, i, oo, c)]
                            assert max(vals) - min(vals) <= 1e-12 * scale, (name, mat, k, o, i, oo, c)


@pytest.mark.parametrize("pk", [67, 330, 25120])
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_orbit_tile_shards_partition(pk, world):
    """Row shard [rlo, rhi) of a block takes orbit tiles [floor(f0 T), floor(f1 T)),
    f = the shard's share of the block's lower triangle (symkr.cuh, curvature.cuh)."""
    T = 3825
    def tri(r):
        j = min(max(r, 0), pk)
        return j * (j + 1.0) / (pk * (pk + 1.0))
    bounds = [round(pk * np.sqrt(s / world)) for s in range(world)] + [pk]
    ranges = []
    for s in range(world):
        f0, f1 = tri(bounds[s]), 1.0 if bounds[s + 1] >= pk else tri(bounds[s + 1])
        t0 = int(np.floor(f0 * T))
        t1 = T if f1 >= 1.0 else max(t0, int(np.floor(f1 * T)))
        ranges.append((t0, t1))
    assert ranges[0][0] == 0 and ranges[-1][1] == T
    assert all(ranges[s][1] == ranges[s + 1][0] for s in range(world - 1))
