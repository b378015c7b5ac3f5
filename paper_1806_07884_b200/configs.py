"""The five BASELINE.json configurations, pinned (seeds, radii, mixtures).

Every input is a pure function of the config name (and an optional point
count / index window), generated on the host by librbg_datagen.so so the GPU
path, the CPU oracle and the bench all see bit-identical arrays.  These are
seeded synthetic stand-ins; BASELINE names no public dataset.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _native


@dataclass(frozen=True)
class Config:
    name: str
    dim: int
    n: int
    m: int
    kernel: str
    alpha: float
    description: str

    @property
    def radius(self) -> float:
        return 1.0 / self.alpha


def _alpha_for(m: int, per_support: float, dim: int) -> float:
    if dim == 2:
        r = math.sqrt(per_support / (math.pi * m))
    else:
        r = (per_support / (m * 4.0 * math.pi / 3.0)) ** (1.0 / 3.0)
    return 1.0 / r


CONFIGS: dict[str, Config] = {
    "cfg1": Config("cfg1", 2, 100_000, 1_000, "wendland-3-1", _alpha_for(1_000, 30, 2),
                   "2D Halton N=1e5, h=Franke; M=1e3 Halton centres; phi31, ~30 centres/support"),
    "cfg2": Config("cfg2", 2, 1_000_000, 10_000, "wendland-3-1", _alpha_for(10_000, 50, 2),
                   "2D uniform N=1e6, h=sin4x cos4y + N(0,0.01); M=1e4 on a 100x100 grid; phi31, ~50/support"),
    "cfg3": Config("cfg3", 3, 4_000_000, 50_000, "wendland-3-2", _alpha_for(50_000, 60, 3),
                   "3D uniform N=4e6, h=exp(-|x-.5|^2/.1)+.5 sin6z; M=5e4 Halton; phi32, ~60/support"),
    "cfg4": Config("cfg4", 2, 20_000_000, 100_000, "wendland-3-1", _alpha_for(100_000, 40, 2),
                   "2D Gaussian mixture N=2e7 (+5% uniform floor), h=6-octave fBm; M=1e5 Halton; phi31, ~40/support"),
    "cfg5": Config("cfg5", 2, 200_000_000, 1_000_000, "wendland-3-1", _alpha_for(1_000_000, 40, 2),
                   "2D Halton N=2e8, h=Franke+N(0,0.001); M=1e6 on a 1000x1000 grid; phi31, ~40/support"),
}

SEEDS = {"cfg2": 2, "cfg3": 3, "cfg4": 4, "cfg5": 5}


def _ptr(a: np.ndarray):
    return a.ctypes.data


def halton(start: int, count: int, dims: int) -> np.ndarray:
    out = np.empty((count, dims), dtype=np.float64)
    _native.datagen().dg_halton(start, count, dims, _ptr(out))
    return out


def grid_refs(nx: int, ny: int, box=(0.0, 0.0, 1.0, 1.0)) -> np.ndarray:
    out = np.empty((nx * ny, 2), dtype=np.float64)
    _native.datagen().dg_grid_refs(*box, nx, ny, _ptr(out))
    return out


def franke(xy: np.ndarray) -> np.ndarray:
    xy = np.ascontiguousarray(xy, dtype=np.float64)
    out = np.empty(len(xy), dtype=np.float64)
    _native.datagen().dg_franke(_ptr(xy), len(xy), _ptr(out))
    return out


def centres(name: str) -> np.ndarray:
    c = CONFIGS[name]
    if name == "cfg1":
        return halton(1, c.m, 2)
    if name == "cfg2":
        return grid_refs(100, 100)
    if name == "cfg3":
        return halton(1, c.m, 3)
    if name == "cfg4":
        return halton(1, c.m, 2)
    if name == "cfg5":
        return grid_refs(1000, 1000)
    raise KeyError(name)


def points(name: str, n: int | None = None, start: int = 0, seed_offset: int = 0):
    """Points [start, start+n) of config `name` and their values h.

    `seed_offset` derives independent point sets (used for weak-scaling
    shards); 0 is the canonical config."""
    c = CONFIGS[name]
    n = c.n if n is None else n
    dg = _native.datagen()
    if name in ("cfg1", "cfg5"):
        xy = halton(1 + start + seed_offset * c.n, n, 2)
        h = franke(xy)
        if name == "cfg5":
            h = _noise_window(SEEDS[name] * 1000 + 1 + seed_offset, start, n, 0.001, h)
        return xy, h
    if name == "cfg2":
        xy = _uniform_window(SEEDS[name] + 7919 * seed_offset, start, n, 2)
        h = np.empty(n)
        dg.dg_sincos(_ptr(xy), n, _ptr(h))
        return xy, _noise_window(SEEDS[name] * 1000 + 1 + seed_offset, start, n, 0.01, h)
    if name == "cfg3":
        xyz = _uniform_window(SEEDS[name] + 7919 * seed_offset, start, n, 3)
        h = np.empty(n)
        dg.dg_bump3(_ptr(xyz), n, _ptr(h))
        return xyz, h
    if name == "cfg4":
        xy = _window(lambda cnt, o: dg.dg_mixture(SEEDS[name] + 7919 * seed_offset, cnt, _ptr(o)), start, n, 2)
        h = np.empty(n)
        dg.dg_fbm(SEEDS[name] * 1000 + 1, _ptr(xy), n, _ptr(h))
        return xy, h
    raise KeyError(name)


def _window(fill, start: int, n: int, dims: int) -> np.ndarray:
    """Generators are pure functions of the index: produce [0, start+n) and slice."""
    full = np.empty((start + n, dims), dtype=np.float64)
    fill(start + n, full)
    return np.ascontiguousarray(full[start:])


def _uniform_window(seed: int, start: int, n: int, dims: int) -> np.ndarray:
    return _window(lambda cnt, o: _native.datagen().dg_uniform(seed, cnt, dims, _ptr(o)), start, n, dims)


def _noise_window(seed: int, start: int, n: int, sigma: float, h: np.ndarray) -> np.ndarray:
    noise = np.zeros(start + n)
    _native.datagen().dg_add_noise(seed, start + n, sigma, _ptr(noise))
    return h + noise[start:]


def _bitrev(k: int, bits: int) -> int:
    return int(format(k, f"0{bits}b")[::-1], 2) if bits else 0


def slab_points(name: str, rank: int, world: int, n: int | None = None):
    """Rank `rank`'s equal-count spatial slab (x in 2-D, z in 3-D) of the one
    point set of config `name` -- the strong-scaling shard of SURVEY 8(e).

    For the Halton configs (cfg1, cfg5) and a power-of-two world the slab is
    generated directly: x = radical_inverse(2, i) lies in [k/W, (k+1)/W) iff
    i mod W == bitreverse(k), so rank k owns the indices W q + bitreverse(k)
    (equal counts within one point, no rank materialises the whole set).
    Otherwise the whole set is generated and split with rbg_partition_slabs.
    `n` restricts the set to the config's first n points (tests)."""
    c = CONFIGS[name]
    total = c.n if n is None else n
    if world == 1:
        return points(name, n=total)
    if name in ("cfg1", "cfg5") and world & (world - 1) == 0:
        bits = world.bit_length() - 1
        r = _bitrev(rank, bits)
        first = r if r > 0 else world  # sequence indices start at 1
        count = (total - first) // world + 1 if first <= total else 0
        xy = np.empty((count, 2))
        _native.datagen().dg_halton_strided(first, world, count, 2, _ptr(xy))
        h = franke(xy)
        if name == "cfg5":  # noise of the point at array position i - 1
            _native.datagen().dg_add_noise_strided(SEEDS[name] * 1000 + 1, first - 1, world, count, 0.001, _ptr(h))
        return xy, h
    from . import distributed
    xy, h = points(name, n=total)
    _, slab = distributed.partition_slabs(xy, world)
    sel = slab == rank
    return np.ascontiguousarray(xy[sel]), np.ascontiguousarray(h[sel])


def window_points(name: str, a: int, b: int):
    """The points of a Halton config (cfg1, cfg5) inside the spatial window
    [0, 2^-a) x [0, 3^-b): exactly the sequence indices that are multiples of
    2^a 3^b (radical_inverse(2, i) < 2^-a iff 2^a | i, same for base 3), at
    the config's full density.  Returns (xy, h)."""
    if name not in ("cfg1", "cfg5"):
        raise KeyError(name)
    c = CONFIGS[name]
    stride = (2 ** a) * (3 ** b)
    count = c.n // stride
    xy = np.empty((count, 2))
    _native.datagen().dg_halton_strided(stride, stride, count, 2, _ptr(xy))
    h = franke(xy)
    if name == "cfg5":
        _native.datagen().dg_add_noise_strided(SEEDS[name] * 1000 + 1, stride - 1, stride, count, 0.001, _ptr(h))
    return xy, h
