"""Seeded synthetic workloads for the five BASELINE.json configurations.

The paper and the reference measure no public dataset; BASELINE.json names
five MLP configurations with synthetic input distributions.  This module
draws them deterministically from a splitmix64 stream (the reference's own
generator, /root/reference/proj/include/curv/rng.hpp:14-19), vectorised in
numpy so a 20000 x 1024 draw takes well under a second.

Glorot-uniform weights follow the reference's init_params
(/root/reference/proj/src/cli.cpp:132-146): W entries are
(2u - 1) * sqrt(6 / (T_in + T_out)) drawn layer by layer in canonical order.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def splitmix64(seed: int, count: int, offset: int = 0) -> np.ndarray:
    """The first `count` outputs of rng.hpp's Rng(seed).next_u64() after
    skipping `offset` draws (counter form: state_i = seed + (i+1)*golden)."""
    with np.errstate(over="ignore"):
        i = np.arange(offset + 1, offset + count + 1, dtype=np.uint64)
        z = np.uint64(seed) + i * _GOLDEN
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def uniform(seed: int, count: int) -> np.ndarray:
    """rng.hpp:22 next_uniform(): (u64 >> 11) * 2^-53, in [0, 1)."""
    return (splitmix64(seed, count) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def normal(seed: int, count: int) -> np.ndarray:
    """rng.cpp:8-20 Box-Muller: pairs (cos, sin) from (1-u1, u2)."""
    npairs = (count + 1) // 2
    u = uniform(seed, 2 * npairs)
    u1 = 1.0 - u[0::2]
    u2 = u[1::2]
    r = np.sqrt(-2.0 * np.log(u1))
    th = 2.0 * np.pi * u2
    out = np.empty(2 * npairs)
    out[0::2] = r * np.cos(th)
    out[1::2] = r * np.sin(th)
    return out[:count]


def param_count(widths) -> int:
    return int(sum(widths[k] * widths[k + 1] + widths[k + 1] for k in range(len(widths) - 1)))


def glorot_params(widths, seed: int, bias: str = "zero") -> np.ndarray:
    P = param_count(widths)
    flat = np.zeros(P)
    nw = sum(widths[k] * widths[k + 1] for k in range(len(widths) - 1))
    u = uniform(seed, nw)
    bn = normal(seed ^ 0xB1A5, P) if bias == "normal" else None
    at = 0
    used = 0
    for k in range(len(widths) - 1):
        tin, tout = widths[k], widths[k + 1]
        r = np.sqrt(6.0 / (tin + tout))
        flat[at:at + tin * tout] = (2.0 * u[used:used + tin * tout] - 1.0) * r
        used += tin * tout
        at += tin * tout
        if bn is not None:  # "biases ~ N(0, 0.01)": variance 0.01
            flat[at:at + tout] = 0.1 * bn[at:at + tout]
        at += tout
    return flat


@dataclass
class Workload:
    name: str
    widths: list
    activation: str
    n: int
    x_dist: str
    bias: str
    seed: int
    dtypes: tuple = ("f32",)
    task: str = "hessian+opg"
    eig_k: int = 0
    oversample: int = 0
    power_iters: int = 0
    note: str = ""
    extra: dict = field(default_factory=dict)

    @property
    def P(self) -> int:
        return param_count(self.widths)

    def draw(self):
        """(params, x, y_onehot, labels) as float64 / int32 numpy arrays."""
        T0, TL = self.widths[0], self.widths[-1]
        params = glorot_params(self.widths, self.seed, self.bias)
        if self.x_dist == "uniform":
            x = uniform(self.seed + 1, self.n * T0)
        else:
            x = normal(self.seed + 1, self.n * T0)
        x = x.reshape(self.n, T0)
        labels = (splitmix64(self.seed + 2, self.n) % np.uint64(TL)).astype(np.int32)
        y = np.zeros((self.n, TL))
        y[np.arange(self.n), labels] = 1.0
        return params, x, y, labels


# BASELINE.json "configs", in order.  P follows the reference's param_count
# (model.cpp:89-95); BASELINE.json's P for configs 2 and 3 (55114, 109514)
# are arithmetic slips of the same formula (55050 and 109386 here).
CONFIGS = {
    "c0": Workload("c0", [4, 8, 3], "sigmoid", 150, "uniform", "zero", 0, ("f64",),
                   note="CPU-runnable oracle case; exact Hessian + OPG 67x67"),
    "c1": Workload("c1", [784, 32, 10], "sigmoid", 1000, "uniform", "normal", 1, ("f32", "f64"),
                   note="full OPG + exact Hessian, 25450 x 25450"),
    "c2": Workload("c2", [784, 64, 64, 10], "tanh", 4096, "normal", "zero", 2, ("f32",),
                   task="hessian", note="exact Hessian via batched HVPs, rows sharded"),
    "c3": Workload("c3", [784, 128, 64, 10], "sigmoid", 10000, "uniform", "zero", 3, ("f32",),
                   task="opg", note="full OPG (~48 GB fp32), row-block sharded"),
    "c4": Workload("c4", [1024, 512, 512, 512, 10], "tanh", 20000, "normal", "zero", 4, ("f32",),
                   task="eig", eig_k=100, oversample=20, power_iters=2,
                   note="top-100 OPG eigenpairs by randomized range finder"),
}
