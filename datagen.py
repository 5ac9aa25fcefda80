"""Seeded synthetic inputs shared by the oracle tests, the CUDA parity tests and bench.py.

This module holds NO arithmetic of the method (no DTW, no envelope, no lower bound); it only
draws series and resolves the integer warping window.  It is the one piece of code both the
oracle side and the CUDA side may use ("Input recipe").

The UCR archive the paper evaluates on (§4) is not available; the five
BASELINE.json configs are stood in for by this generator (reading C18):

1. class prototypes  P[c] = cumsum(N(0,1)^L);
2. instance n has class n mod C, then a seeded permutation of the instances;
3. a smooth monotone time warp tau(t) = clip(t + m*g(t), 0, L-1) made monotone by a running
   max, g = sum_{r=1,2} a_r sin(2 pi f_r t / L + phi_r), f_r ~ U(0.5,2), phi_r ~ U(0,2 pi),
   a_r ~ N(0,1), rescaled so max|g| = U(0,1); m = shift * L;
4. x = interp(tau; P[c]) + sigma * N(0,1)^L, z-normalised (mean 0, population std 1), float32.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

SEED_BASE = 180809617 * 10


def window_from_percent(p: int, L: int) -> int:
    """Integer warping window w = min(L-1, ceil(p*L/100)) in exact integer arithmetic.

    Reading C4: the paper gives windows as fractions of L (PAPER.md l.563-565,
    "W={0.1*L,0.2*L,...,L}") and is silent on rounding; float ceil(0.07*300) would give 22.
    """
    if p < 0 or L < 1:
        raise ValueError("p must be >= 0 and L >= 1")
    return min(L - 1, (p * L + 99) // 100)


@dataclass(frozen=True)
class Config:
    idx: int
    name: str
    n_train: int
    n_test: int          # 0 for the LOOCV config (leave-one-out over the train set)
    L: int
    classes: int
    shift: float         # maximum warp as a fraction of L
    sigma: float         # noise std
    percents: tuple      # window grid in percent of L
    Vs: tuple            # tightness parameters
    extra: dict = field(default_factory=dict)

    def windows(self) -> list[int]:
        return [window_from_percent(p, self.L) for p in self.percents]


# BASELINE.json "configs" (cited as BJ:configs[k]).
CONFIGS = {
    0: Config(0, "tiny", 100, 100, 128, 5, 0.05, 0.1, (10,), (5,)),
    1: Config(1, "paper_like_pairs", 1000, 1000, 256, 10, 0.10, 0.1,
              (1, 10, 20, 50, 100), (1, 2, 4, 5, 8)),
    2: Config(2, "large_search", 100_000, 10_000, 512, 20, 0.05, 0.1, (20,), (5,)),
    3: Config(3, "loocv_window_search", 2000, 0, 300, 8, 0.05, 0.1, tuple(range(101)), (5,)),
    4: Config(4, "long_full_window", 10_000, 1000, 2048, 4, 0.20, 0.2, (100,), (8,)),
}


def _warp_indices(rng: np.random.Generator, n: int, L: int, m: float) -> np.ndarray:
    t = np.arange(L, dtype=np.float64)[None, :]
    f = rng.uniform(0.5, 2.0, size=(n, 2))
    phi = rng.uniform(0.0, 2.0 * np.pi, size=(n, 2))
    a = rng.standard_normal(size=(n, 2))
    g = (a[:, 0:1] * np.sin(2.0 * np.pi * f[:, 0:1] * t / L + phi[:, 0:1])
         + a[:, 1:2] * np.sin(2.0 * np.pi * f[:, 1:2] * t / L + phi[:, 1:2]))
    gmax = np.max(np.abs(g), axis=1, keepdims=True)
    gmax[gmax == 0.0] = 1.0
    target = rng.uniform(0.0, 1.0, size=(n, 1))
    g = g / gmax * target
    tau = np.clip(t + m * g, 0.0, L - 1.0)
    return np.maximum.accumulate(tau, axis=1)


def _instances(rng: np.random.Generator, protos: np.ndarray, n: int, shift: float,
               sigma: float, chunk: int = 8192) -> tuple[np.ndarray, np.ndarray]:
    C, L = protos.shape
    labels = (np.arange(n) % C).astype(np.int32)
    labels = labels[rng.permutation(n)]
    out = np.empty((n, L), dtype=np.float32)
    m = shift * L
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        lab = labels[s:e]
        tau = _warp_indices(rng, e - s, L, m)
        lo = np.floor(tau).astype(np.int64)
        lo = np.minimum(lo, L - 1)
        hi = np.minimum(lo + 1, L - 1)
        fr = tau - lo
        p = protos[lab]
        x = (np.take_along_axis(p, lo, axis=1) * (1.0 - fr)
             + np.take_along_axis(p, hi, axis=1) * fr)
        x = x + sigma * rng.standard_normal(size=x.shape)
        mu = x.mean(axis=1, keepdims=True)
        sd = x.std(axis=1, keepdims=True)
        sd[sd == 0.0] = 1.0
        out[s:e] = ((x - mu) / sd).astype(np.float32)
    return out, labels


@dataclass
class Dataset:
    cfg: Config
    train: np.ndarray        # float32 [N][L]
    train_labels: np.ndarray  # int32 [N]
    test: np.ndarray         # float32 [Q][L] (empty for LOOCV)
    test_labels: np.ndarray  # int32 [Q]


def make_dataset(cfg_idx: int, n_train: int | None = None, n_test: int | None = None,
                 seed_offset: int = 0) -> Dataset:
    """Deterministic dataset for BASELINE.json config `cfg_idx`.

    `n_train`/`n_test` truncate the generated sets (a prefix of the full-size draw is NOT
    guaranteed; a reduced draw is its own seeded dataset with the same recipe and shapes).
    """
    cfg = CONFIGS[cfg_idx]
    N = cfg.n_train if n_train is None else n_train
    Q = cfg.n_test if n_test is None else n_test
    ss = np.random.SeedSequence(SEED_BASE + cfg.idx + 1000 * seed_offset)
    s_proto, s_train, s_test = ss.spawn(3)
    rp = np.random.Generator(np.random.PCG64(s_proto))
    protos = np.cumsum(rp.standard_normal(size=(cfg.classes, cfg.L)), axis=1)
    tr, trl = _instances(np.random.Generator(np.random.PCG64(s_train)), protos, N,
                         cfg.shift, cfg.sigma)
    if Q > 0:
        te, tel = _instances(np.random.Generator(np.random.PCG64(s_test)), protos, Q,
                             cfg.shift, cfg.sigma)
    else:
        te = np.empty((0, cfg.L), dtype=np.float32)
        tel = np.empty((0,), dtype=np.int32)
    return Dataset(cfg, tr, trl, te, tel)


def random_series(rng: np.random.Generator, n: int, L: int, kind: str = "walk") -> np.ndarray:
    """Small adversarial inputs for parity/edge tests: random walks, i.i.d. normals, small
    integer grids (many exact ties), or constant series."""
    if kind == "walk":
        x = np.cumsum(rng.standard_normal(size=(n, L)), axis=1)
    elif kind == "normal":
        x = rng.standard_normal(size=(n, L))
    elif kind == "int":
        x = rng.integers(-3, 4, size=(n, L)).astype(np.float64)
    elif kind == "const":
        x = np.repeat(rng.standard_normal(size=(n, 1)), L, axis=1)
    else:
        raise ValueError(kind)
    return np.ascontiguousarray(x.astype(np.float32))
