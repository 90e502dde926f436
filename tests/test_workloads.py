"""Seeded workload generator (paper_1905_05559_b200.workloads)."""
import numpy as np

from paper_1905_05559_b200 import workloads as W


def test_splitmix64_known_answer():
    # splitmix64 with seed 0: published first outputs
    z = W.splitmix64(0, 3)
    assert [int(v) for v in z] == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]


def test_uniform_and_normal_ranges():
    u = W.uniform(7, 10000)
    assert u.min() >= 0.0 and u.max() < 1.0
    g = W.normal(7, 20000)
    assert abs(g.mean()) < 0.05 and abs(g.std() - 1.0) < 0.05


def test_configs_param_counts():
    assert W.CONFIGS["c0"].P == 67
    assert W.CONFIGS["c1"].P == 25450
    assert W.CONFIGS["c4"].P == 1055242
    # reference formula (model.cpp:89-95); BASELINE.json's 55114 / 109514 are slips
    assert W.CONFIGS["c2"].P == 55050
    assert W.CONFIGS["c3"].P == 109386


def test_draw_is_deterministic_and_one_hot():
    a = W.CONFIGS["c0"].draw()
    b = W.CONFIGS["c0"].draw()
    for u, v in zip(a, b):
        assert np.array_equal(u, v)
    p, x, y, lab = a
    assert np.all(y.sum(1) == 1.0) and np.all(y[np.arange(len(lab)), lab] == 1.0)
    assert x.min() >= 0.0 and x.max() < 1.0  # U(0,1) for config 0
    widths = W.CONFIGS["c0"].widths
    r = np.sqrt(6.0 / (widths[0] + widths[1]))
    assert np.abs(p[:32]).max() <= r and np.all(p[32:40] == 0.0)  # Glorot W, zero biases
