"""Binary CSR cache of the BASELINE.json configurations.

Configs 4-5 have 10^8-10^9 entries: generating them costs tens of seconds of host
time per process, and Matrix Market text would be ~20 GB. The standalone writer
lib/f3rg_gen (csrc/problem_gen.cpp + csrc/problems.cpp, host code only) writes
the scaled system once per host into F3RG_CACHE_DIR (default /tmp/f3rg_cache);
readers memory-map it:

    p = load(5)          # p.n, p.nnz, p.row_ptr, p.col_idx, p.values, p.b

This module never loads libf3rg.so, so a process can use it to feed the
UNMODIFIED reference without mapping the product library (bench.py's reference
arm). The bytes are identical to problems.problem(config)'s (tests/test_problems.py).
"""
from __future__ import annotations

import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
GEN = os.path.join(_HERE, "lib", "f3rg_gen")
MAGIC = b"F3RGCSR1"

# config -> (generator kind, default grid, param, pattern seed, rhs mode, rhs seed);
# the same table as problems.CONFIGS (checked by tests/test_problems.py)
CONFIGS = {
    1: (1, (64, 64, 64), 0.0, 0, 0, 0),
    2: (2, (128, 128, 128), 0.0, 0, 0, 1),
    3: (3, (192, 192, 192), 0.0, 0, 0, 2),
    4: (4, (256, 256, 256), 0.0, 3, 1, 0),
    5: (5, (20_000_000, 0, 0), 0.0, 4, 0, 4),
}


@dataclass
class CachedProblem:
    name: str
    n: int
    row_ptr: np.ndarray
    col_idx: np.ndarray
    values: np.ndarray
    b: np.ndarray
    path: str

    @property
    def nnz(self) -> int:
        return int(self.col_idx.size)


def cache_dir() -> str:
    return os.environ.get("F3RG_CACHE_DIR", "/tmp/f3rg_cache")


def _grid(config: int, grid):
    kind, dgrid = CONFIGS[config][0], CONFIGS[config][1]
    if grid is None:
        return tuple(dgrid)
    if isinstance(grid, int):
        return (grid, 0, 0) if kind == 5 else (grid, grid, grid)
    return tuple(list(grid) + [0, 0])[:3]


def cache_path(config: int, grid=None) -> str:
    g = _grid(config, grid)
    return os.path.join(cache_dir(), f"config{config}_{'x'.join(str(v) for v in g if v)}.csr")


def ensure(config: int, grid=None) -> str:
    """path of the cache file, writing it with lib/f3rg_gen first if absent"""
    path = cache_path(config, grid)
    if os.path.exists(path):
        return path
    if not os.path.exists(GEN):
        raise FileNotFoundError(f"{GEN} is missing: run `python -m paper_2505_20719_b200.buildlib`")
    os.makedirs(os.path.dirname(path), exist_ok=True)
    kind, _, param, seed, mode, rseed = CONFIGS[config]
    g = _grid(config, grid)
    subprocess.run([GEN, str(kind), *(str(v) for v in g), repr(param), str(seed), str(mode), str(rseed), path],
                   check=True)
    return path


def load(config: int, grid=None) -> CachedProblem:
    path = ensure(config, grid)
    with open(path, "rb") as f:
        head = f.read(24)
    if head[:8] != MAGIC:
        raise ValueError(f"{path}: not an F3RGCSR1 file")
    n, nnz = (int(v) for v in np.frombuffer(head[8:24], dtype=np.uint64))
    off = 24
    arrays = []
    for dt, count in ((np.uint32, n + 1), (np.uint32, nnz), (np.float64, nnz), (np.float64, n)):
        arrays.append(np.memmap(path, dtype=dt, mode="r", offset=off, shape=(count,)))
        off += count * np.dtype(dt).itemsize
    if off != os.path.getsize(path):
        raise ValueError(f"{path}: size {os.path.getsize(path)} != {off}")
    rp, ci, val, b = arrays
    g = _grid(config, grid)
    name = f"config{config}" + ("" if g == tuple(CONFIGS[config][1]) else "@" + "x".join(str(v) for v in g if v))
    return CachedProblem(name, n, rp, ci, val, b, path)
