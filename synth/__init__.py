"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NO arithmetic of the Falkon method (no kernel, no solver, no
preconditioner): it only draws the data the method is run on.  Both the oracle
(``oracle/``) and the CUDA path (``paper_2006_10350_b200``) receive the arrays it
returns; neither side imports the other.

Recipe:
  * X ~ N(0, 1) i.i.d., rounded to fp32.  The paper's datasets are standardised to
    zero mean / unit variance (App. A.3), so i.i.d. standard normal
    features reproduce the value distribution; the shapes (n, d) come from
    BASELINE.json and Table 3.
  * y = sin(x_1 + x_2 + x_3) + 0.3 * N(0, 1)  (regression configs), or its sign
    (binary / single-column classification configs: TIMIT, HIGGS).
  * Centers C: m rows of X drawn uniformly WITHOUT replacement
    ("sampled uniformly at random"; SURVEY.md reading c11).
  * Every element is a pure function of (seed, stream, row, column): a
    splitmix64 hash of the element's global index feeds a Box-Muller transform.
    Any row range (a GPU shard, an oracle prefix, one row) can therefore be
    regenerated independently and bit-identically.
"""
from __future__ import annotations

import dataclasses
import numpy as np

__all__ = ["Config", "CONFIGS", "gen_rows", "gen_X", "gen_y", "center_indices",
           "gen_C", "gen_vec", "make_problem", "shard_range"]

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)
_GOLD = np.uint64(0x9E3779B97F4A7C15)
_C1 = np.uint64(0xBF58476D1CE4E5B9)
_C2 = np.uint64(0x94D049BB133111EB)

# stream ids: independent sub-sequences per array
STREAM_X = 1
STREAM_NOISE = 2
STREAM_VEC = 3
STREAM_XTEST = 4


@dataclasses.dataclass(frozen=True)
class Config:
    """One BASELINE.json configuration.  sigma/lam/iters from Table 3
    where BASELINE.json is silent."""
    name: str
    n: int
    d: int
    m: int
    sigma: float
    lam: float
    iters: int
    seed: int
    task: str  # "reg" | "cls"


CONFIGS = {
    # BASELINE.json configs[0..4]
    "tiny": Config("tiny", 2_000, 8, 100, 1.0, 1e-6, 10, 0, "reg"),
    "msd": Config("msd", 463_715, 90, 50_000, 7.0, 2e-6, 20, 1, "reg"),
    "timit": Config("timit", 1_100_000, 440, 100_000, 14.5, 5e-9, 5, 2, "cls"),
    "higgs": Config("higgs", 10_500_000, 28, 100_000, 3.8, 3e-8, 10, 3, "cls"),
    "taxi": Config("taxi", 1_000_000_000, 9, 50_000, 1.0, 2e-7, 7, 4, "reg"),
}


@dataclasses.dataclass(frozen=True)
class GscConfig:
    """LogFalkon (Alg. 2) workloads: Table 3 LogFalkon column for HIGGS
    (m = 1e5, sigma = 5, lambda = 1e-9, 9 Newton steps) and a tiny case for the CPU oracle.
    The level path is explicit (reading g5): geometric from mus[0] to lambda."""
    name: str
    base: str          # Config supplying n, d, seed and the +-1 labels
    m: int
    sigma: float
    mus: tuple
    iters: tuple


def _geom(hi: float, lo: float, k: int) -> tuple:
    return tuple(float(hi * (lo / hi) ** (i / (k - 1))) for i in range(k))


GSC_CONFIGS = {
    "tiny_log": GscConfig("tiny_log", "tiny", 100, 1.0, _geom(1e-2, 1e-6, 5), (5, 5, 5, 5, 10)),
    "higgs_log": GscConfig("higgs_log", "higgs", 100_000, 5.0, _geom(1e-3, 1e-9, 9),
                           (5,) * 8 + (10,)),
}


def make_gsc_problem(name: str, n: int | None = None, m: int | None = None):
    """(gcfg, X, y, C, yC): +-1 labels (cls task of the base config), C = m rows of X and
    yC = their labels (the y_m of Alg. 2)."""
    g = GSC_CONFIGS[name]
    base = CONFIGS[g.base]
    nn = base.n if n is None else n
    mm = g.m if m is None else m
    X = gen_X(base.seed, 0, nn, base.d)
    y = gen_y(base.seed, X, 0, "cls")
    idx = center_indices(base.seed, nn, mm)
    return g, X, y, X[idx].copy(), y[idx].copy()

def _splitmix64(z: np.ndarray) -> np.ndarray:
    z = (z + _GOLD) & _M64
    z = ((z ^ (z >> np.uint64(30))) * _C1) & _M64
    z = ((z ^ (z >> np.uint64(27))) * _C2) & _M64
    return z ^ (z >> np.uint64(31))


def _normals(seed: int, stream: int, index: np.ndarray) -> np.ndarray:
    """Standard normals (fp64) as a pure function of (seed, stream, global index)."""
    key = np.uint64((seed * 0x100000001B3 + stream * 0x5851F42D4C957F2D) & 0xFFFFFFFFFFFFFFFF)
    with np.errstate(over="ignore"):
        h = _splitmix64(_splitmix64(index.astype(np.uint64) ^ key))
    u1 = ((h >> np.uint64(32)).astype(np.float64) + 1.0) / 4294967296.0  # (0, 1]
    u2 = (h & np.uint64(0xFFFFFFFF)).astype(np.float64) / 4294967296.0   # [0, 1)
    return np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)


def gen_rows(seed: int, stream: int, rows: np.ndarray, d: int) -> np.ndarray:
    """fp32 matrix whose row r is the generator's row rows[r] (any order, any subset)."""
    rows = np.asarray(rows, dtype=np.int64)
    out = np.empty((rows.size, d), dtype=np.float32)
    step = max(1, (1 << 22) // max(d, 1))
    cols = np.arange(d, dtype=np.int64)
    for s in range(0, rows.size, step):
        r = rows[s:s + step]
        idx = r[:, None] * d + cols[None, :]
        out[s:s + step] = _normals(seed, stream, idx).astype(np.float32)
    return out


def gen_X(cfg_or_seed, row0: int = 0, nrows: int | None = None, d: int | None = None,
          stream: int = STREAM_X) -> np.ndarray:
    """Rows [row0, row0+nrows) of X (fp32, row-major)."""
    if isinstance(cfg_or_seed, Config):
        seed, d = cfg_or_seed.seed, cfg_or_seed.d
        if nrows is None:
            nrows = cfg_or_seed.n - row0
    else:
        seed = int(cfg_or_seed)
    return gen_rows(seed, stream, np.arange(row0, row0 + nrows, dtype=np.int64), d)


def gen_y(seed: int, X: np.ndarray, row0: int, task: str = "reg") -> np.ndarray:
    """Targets for rows [row0, row0+len(X)) (fp32)."""
    noise = _normals(seed, STREAM_NOISE, np.arange(row0, row0 + X.shape[0], dtype=np.int64))
    k = min(3, X.shape[1])
    y = np.sin(X[:, :k].astype(np.float64).sum(axis=1)) + 0.3 * noise
    if task == "cls":
        y = np.where(y >= 0.0, 1.0, -1.0)
    return y.astype(np.float32)


def gen_y_rows(seed: int, X: np.ndarray, rows: np.ndarray, task: str = "reg") -> np.ndarray:
    """Targets of the generator rows `rows` (any subset, e.g. the centres' y_m) given those
    rows' X; equals gen_y on a contiguous range."""
    noise = _normals(seed, STREAM_NOISE, np.asarray(rows, dtype=np.int64))
    k = min(3, X.shape[1])
    y = np.sin(X[:, :k].astype(np.float64).sum(axis=1)) + 0.3 * noise
    if task == "cls":
        y = np.where(y >= 0.0, 1.0, -1.0)
    return y.astype(np.float32)


def center_indices(seed: int, n: int, m: int) -> np.ndarray:
    """m distinct row indices drawn uniformly without replacement, sorted."""
    rng = np.random.Generator(np.random.PCG64(seed + 7919))
    idx = rng.choice(n, size=m, replace=False)
    return np.sort(idx.astype(np.int64))


def gen_C(seed: int, n: int, m: int, d: int) -> np.ndarray:
    return gen_rows(seed, STREAM_X, center_indices(seed, n, m), d)


def gen_vec(seed: int, m: int, stream: int = STREAM_VEC) -> np.ndarray:
    """Benchmark / parity vector v ~ N(0,1), fp32 (seed 100+cfg)."""
    return _normals(seed + 100, stream, np.arange(m, dtype=np.int64)).astype(np.float32)


def shard_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous row block of rank `rank`: first n % world ranks get one more row."""
    base, extra = divmod(n, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def make_problem(name_or_cfg, n: int | None = None, m: int | None = None,
                 row0: int = 0):
    """(cfg, X, y, C) for a config, optionally on a row subrange (n rows from row0)
    and/or fewer centers.  Centers are m rows of the generated X (C subset of X)."""
    cfg = CONFIGS[name_or_cfg] if isinstance(name_or_cfg, str) else name_or_cfg
    nn = cfg.n if n is None else n
    mm = cfg.m if m is None else m
    X = gen_X(cfg.seed, row0, nn, cfg.d)
    y = gen_y(cfg.seed, X, row0, cfg.task)
    C = gen_rows(cfg.seed, STREAM_X, row0 + center_indices(cfg.seed, nn, mm), cfg.d)
    return cfg, X, y, C


# ---------------------------------------------------------------------------------------
# Device-side generation (torch) of the same stream, for inputs too large to build on the
# host (TAXI: 1e9 x 9).  Same splitmix64 hash and Box-Muller; uint64 arithmetic is emulated
# on int64 (wrapping multiply, masked logical shifts).  The fp64 log/cos of the device may
# differ from NumPy's in the last ulp, so a few fp32 values can differ by one ulp from
# gen_X; tests that compare against the oracle read the rows back from the device tensor.
def _t_splitmix64(z):
    import torch
    gold = torch.tensor(0x9E3779B97F4A7C15 - (1 << 64), dtype=torch.int64, device=z.device)
    c1 = torch.tensor(0xBF58476D1CE4E5B9 - (1 << 64), dtype=torch.int64, device=z.device)
    c2 = torch.tensor(0x94D049BB133111EB - (1 << 64), dtype=torch.int64, device=z.device)

    def srl(x, s):  # logical right shift on int64
        return (x >> s) & ((1 << (64 - s)) - 1)

    z = z + gold
    z = (z ^ srl(z, 30)) * c1
    z = (z ^ srl(z, 27)) * c2
    return z ^ srl(z, 31)


def gen_X_torch(seed: int, row0: int, nrows: int, d: int, device="cuda", stream: int = STREAM_X,
                chunk_rows: int = 1 << 22):
    """fp32 tensor (nrows x d) on `device` with rows [row0, row0+nrows) of the generator."""
    import torch
    key = (seed * 0x100000001B3 + stream * 0x5851F42D4C957F2D) & 0xFFFFFFFFFFFFFFFF
    if key >= 1 << 63:
        key -= 1 << 64
    out = torch.empty((nrows, d), dtype=torch.float32, device=device)
    cols = torch.arange(d, dtype=torch.int64, device=device)
    for s in range(0, nrows, chunk_rows):
        r = torch.arange(row0 + s, row0 + min(nrows, s + chunk_rows), dtype=torch.int64,
                         device=device)
        idx = r[:, None] * d + cols[None, :]
        h = _t_splitmix64(_t_splitmix64(idx ^ key))
        u1 = (((h >> 32) & 0xFFFFFFFF).to(torch.float64) + 1.0) / 4294967296.0
        u2 = (h & 0xFFFFFFFF).to(torch.float64) / 4294967296.0
        out[s:s + r.numel()] = (torch.sqrt(-2.0 * torch.log(u1)) *
                                torch.cos(2.0 * torch.pi * u2)).to(torch.float32)
    return out


def _t_normals(seed: int, stream: int, index):
    """Device version of _normals (same hash and Box-Muller, fp64)."""
    import torch
    key = (seed * 0x100000001B3 + stream * 0x5851F42D4C957F2D) & 0xFFFFFFFFFFFFFFFF
    if key >= 1 << 63:
        key -= 1 << 64
    h = _t_splitmix64(_t_splitmix64(index ^ key))
    u1 = (((h >> 32) & 0xFFFFFFFF).to(torch.float64) + 1.0) / 4294967296.0
    u2 = (h & 0xFFFFFFFF).to(torch.float64) / 4294967296.0
    return torch.sqrt(-2.0 * torch.log(u1)) * torch.cos(2.0 * torch.pi * u2)


def gen_y_torch(seed: int, X, row0: int, task: str = "reg", chunk_rows: int = 1 << 24):
    """Device version of gen_y for a device-resident X (rows [row0, row0+len(X)))."""
    import torch
    n = X.shape[0]
    k = min(3, X.shape[1])
    y = torch.empty(n, dtype=torch.float32, device=X.device)
    for s in range(0, n, chunk_rows):
        e = min(n, s + chunk_rows)
        r = torch.arange(row0 + s, row0 + e, dtype=torch.int64, device=X.device)
        v = torch.sin(X[s:e, :k].to(torch.float64).sum(dim=1)) + 0.3 * _t_normals(seed, STREAM_NOISE, r)
        if task == "cls":
            v = torch.where(v >= 0.0, 1.0, -1.0)
        y[s:e] = v.to(torch.float32)
    return y
