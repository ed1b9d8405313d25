"""Seeded synthetic inputs for the five BASELINE.json configs.

The paper's ClueWeb09-B posting lists are unavailable; these
counter-based (splitmix64) generators stand in with the configs' shapes, sizes
and value distributions.  Implemented in C (csrc/svb_gen.c, libsvbgen.so) so
2^28..2^31-element inputs generate in seconds on all host cores.

This module loads ONLY the generator library (never the codec library), and has
no package-relative imports, so bench.py's CPU reference arm can load it as a
standalone file without mapping libbytecodec_b200.so.  Every generator has a
shard form (``*_range``) that produces exactly the elements / lists one rank
owns, identical to the same part of the whole-config output.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from pathlib import Path

import numpy as np

GEN_PATH = Path(__file__).resolve().parent / "lib" / "libsvbgen.so"
if not GEN_PATH.exists():
    raise ImportError(f"{GEN_PATH} not found: build it with `make` at the repo root")
_gen = C.CDLL(str(GEN_PATH))
_vp, _u32, _u64, _int = C.c_void_p, C.c_uint32, C.c_uint64, C.c_int
for _name, (_res, _args) in {
    "svbgen_splitmix64": (_u64, [_u64, _u64]),
    "svbgen_uniform_classes": (None, [_u64, _u64, _vp, _int]),
    "svbgen_geometric_sorted": (None, [_u64, _u64, C.c_double, _u32, _vp, _int]),
    "svbgen_geometric_sorted_range": (None, [_u64, _u64, _u64, C.c_double, _vp, _int]),
    "svbgen_list_lengths": (_u64, [_u64, _u64, _u64, _vp]),
    "svbgen_posting_lists": (None, [_u64, _u64, _vp, _vp, _u32, _vp, _int]),
    "svbgen_posting_lists_range": (None, [_u64, _u64, _u64, _vp, _vp, _u32, _vp, _int]),
}.items():
    _fn = getattr(_gen, _name)
    _fn.restype, _fn.argtypes = _res, _args

SEEDS = {1: 0x5EB1_0001, 2: 0x5EB1_0002, 3: 0x5EB1_0003, 4: 0x5EB1_0004, 5: 0x5EB1_0005}


def _threads() -> int:
    return max(1, min(64, os.cpu_count() or 1))


def splitmix64(seed: int, i: int) -> int:
    return int(_gen.svbgen_splitmix64(seed, i))


def uniform_classes(n: int, seed: int) -> np.ndarray:
    """Configs 1/3: byte length i.i.d. uniform over {1,2,3,4}, value uniform in that length's range."""
    out = np.empty(n, np.uint32)
    _gen.svbgen_uniform_classes(seed, n, out.ctypes.data, _threads())
    return out


def geometric_sorted(n: int, mean_gap: float, seed: int, start: int = 0) -> np.ndarray:
    """Configs 2/5: x_0 = start, x_i = x_{i-1} + g_i, g_i geometric on {1,2,..} with the given mean (mod 2^32)."""
    out = np.empty(n, np.uint32)
    _gen.svbgen_geometric_sorted(seed, n, float(mean_gap), start, out.ctypes.data, _threads())
    return out


def geometric_sorted_range(i0: int, n: int, mean_gap: float, seed: int) -> np.ndarray:
    """Elements [i0, i0 + n) of geometric_sorted(N, mean_gap, seed) (start 0), without the ones before."""
    out = np.empty(n, np.uint32)
    _gen.svbgen_geometric_sorted_range(seed, i0, n, float(mean_gap), out.ctypes.data, _threads())
    return out


@dataclass
class ListBatch:
    values: np.ndarray   # concatenated lists (uint32)
    lengths: np.ndarray  # per list (uint32)
    offsets: np.ndarray  # element offset of each list (uint64), len = nlists + 1
    cap: int             # water-fill cap applied to the lengths


def list_lengths(nlists: int, seed: int, cap_total: int = 1 << 30) -> tuple[np.ndarray, int]:
    """Config 4 list lengths: L_i = floor(2^U), U ~ U(4,16), water-fill capped to cap_total."""
    lens = np.empty(nlists, np.uint32)
    cap = int(_gen.svbgen_list_lengths(seed, nlists, cap_total, lens.ctypes.data))
    return lens, cap


def posting_lists(nlists: int, seed: int, cap_total: int = 1 << 30, universe: int = 1 << 25) -> ListBatch:
    """Config 4: L_i = floor(2^U), U ~ U(4,16), water-fill capped to cap_total in total; each list
    strictly increasing in [0, universe)."""
    lens, cap = list_lengths(nlists, seed, cap_total)
    offs = np.zeros(nlists + 1, np.uint64)
    np.cumsum(lens, out=offs[1:])
    vals = np.empty(int(offs[-1]), np.uint32)
    _gen.svbgen_posting_lists(seed, nlists, lens.ctypes.data, offs.ctypes.data, universe, vals.ctypes.data,
                              _threads())
    return ListBatch(vals, lens, offs, cap)


def posting_lists_range(lens_all: np.ndarray, l0: int, l1: int, seed: int, universe: int = 1 << 25) -> ListBatch:
    """Lists [l0, l1) of posting_lists (same lengths array), generated alone: one rank's shard."""
    lens = np.ascontiguousarray(lens_all[l0:l1], np.uint32)
    offs = np.zeros(lens.size + 1, np.uint64)
    np.cumsum(lens, out=offs[1:])
    vals = np.empty(int(offs[-1]), np.uint32)
    if lens.size:
        _gen.svbgen_posting_lists_range(seed, l0, lens.size, lens.ctypes.data, offs.ctypes.data, universe,
                                        vals.ctypes.data, _threads())
    return ListBatch(vals, lens, offs, 0)


# Full BASELINE.json sizes
CONFIG_N = {1: 1 << 20, 2: 1 << 26, 3: 1 << 28, 4: 1 << 20, 5: 1 << 31}
CFG5_CHUNK = 1 << 16


def config_array(cfg: int, n: int | None = None) -> np.ndarray:
    """Single-array input of config 1, 2, 3 or 5 (n overrides the size for scaled-down parity cases)."""
    n = CONFIG_N[cfg] if n is None else n
    if cfg in (1, 3):
        return uniform_classes(n, SEEDS[cfg])
    if cfg == 2:
        return geometric_sorted(n, 8.0, SEEDS[2])
    if cfg == 5:
        return geometric_sorted(n, 32.0, SEEDS[5])
    raise ValueError(f"config {cfg} is not a single array")
