"""Version-independent synthetic inputs for the parity tests and goldens.

Values come from splitmix64 (pure uint64 arithmetic, no library RNG whose
algorithm could change between numpy versions), mapped to uniform floats and
rounded to fp32, so the device (fp32) and the oracle / reference (fp64
upcasts) see exactly the same numbers.
"""

import numpy as np

M = np.uint64(0xFFFFFFFFFFFFFFFF)


def _splitmix64(seed, n):
    with np.errstate(over="ignore"):
        idx = np.arange(1, n + 1, dtype=np.uint64)
        z = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) + idx * np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z


def uniform(seed, n, lo, hi):
    """n fp32 values ~ U(lo, hi) (53-bit uniform, then rounded to fp32)."""
    u = (_splitmix64(seed, n) >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)
    return (lo + (hi - lo) * u).astype(np.float32)


def layout_numel(layout):
    out = []
    for _, shape, _ in layout:
        n = 1
        for d in shape:
            n *= d
        out.append(n)
    return out


def group_inputs(layout, seed, *, w_scale=0.05, g_scale=1e-3, m_scale=1e-4, zero_w=(), zero_g=()):
    """Per-group fp32 (w, g, m) arrays, shapes from the layout."""
    out = []
    for i, ((name, shape, cat), n) in enumerate(zip(layout, layout_numel(layout))):
        w = uniform(seed * 1000003 + 3 * i, n, -w_scale, w_scale)
        g = uniform(seed * 1000003 + 3 * i + 1, n, -g_scale, g_scale)
        m = uniform(seed * 1000003 + 3 * i + 2, n, -m_scale, m_scale)
        if cat == "norm-scale":
            w = (w + np.float32(1.0)).astype(np.float32)
        if name in zero_w:
            w[:] = 0
        if name in zero_g:
            g[:] = 0
        out.append((w.reshape(shape), g.reshape(shape), m.reshape(shape)))
    return out


def step_grads(layout, seed, step, g_scale=1e-3):
    """Fresh gradient per step t for trajectory tests."""
    return [uniform(seed * 7919 + step * 1000003 + i, n, -g_scale, g_scale).reshape(shape)
            for i, ((_, shape, _), n) in enumerate(zip(layout, layout_numel(layout)))]


RAGGED = [
    ("a.weight", (3, 5), "weight"),
    ("a.bias", (5,), "bias"),
    ("b.weight", (33, 7), "weight"),
    ("bn.scale", (7,), "norm-scale"),
    ("bn.shift", (7,), "norm-shift"),
    ("c.weight", (129,), "weight"),
    ("one.weight", (1,), "weight"),
    ("zero.weight", (40,), "weight"),
    ("nograd.weight", (17,), "weight"),
    ("big.weight", (1000, 3), "weight"),
    ("big.bias", (3,), "bias"),
]
