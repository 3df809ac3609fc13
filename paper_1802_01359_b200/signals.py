"""Seeded synthetic input generators for the five BASELINE.json configs.

This module holds NONE of the method's arithmetic: it only draws signals.  It
is the one module shared by the oracle-side tests and the CUDA-side tests and
bench.  The paper uses no public dataset
(PAPER.md:693 mentions only an unnamed "vector of tenths of millions of
points"); these recipes stand in for it, shaped as BASELINE.json configs 0-4.

RNG: numpy PCG64 via default_rng(SeedSequence([cfg, i, t])) for signal i,
sub-seed t (t > 0 only when a parity test screens a seed).  Grid x_j = j/n
(periodic, reading A11).  "log-uniform integer in [a, b]" =
min(b, floor(exp(U(ln a, ln(b+1))))).  Draws run in the order written; the
noise is drawn last as one standard_normal(n) call.
"""
from __future__ import annotations

import math

import numpy as np

TWO_PI = 2.0 * math.pi

# name -> (n, batch, dtype, delta) ; xi = 1.6, max_inner = 200, max_imfs = 10 for all
CONFIGS = {
    "cfg0": dict(n=1024, batch=1, dtype="f64", delta=1e-3),
    "cfg1": dict(n=4096, batch=4096, dtype="f64", delta=1e-3),
    "cfg2": dict(n=65536, batch=512, dtype="f64", delta=1e-4),
    "cfg3": dict(n=1 << 26, batch=1, dtype="f64", delta=1e-3),
}
CFG4_LENGTHS = [1 << 10, 1 << 14, 1 << 17, 1 << 20, 3 << 14, 5 << 14]
CFG_INDEX = {"cfg0": 0, "cfg1": 1, "cfg2": 2, "cfg3": 3, "cfg4": 4}
XI, MAX_INNER, MAX_IMFS = 1.6, 200, 10


def cfg4_batch(n: int) -> int:
    """fp32 sweep: batch fills 1 GiB (2^28 fp32 samples) per run."""
    return (1 << 28) // n


def _rng(cfg: int, i: int, t: int = 0) -> np.random.Generator:
    return np.random.default_rng(np.random.SeedSequence([cfg, i, t]))


def _loguniform_int(rng, a: int, b: int, size=None):
    u = rng.uniform(math.log(a), math.log(b + 1), size)
    return np.minimum(b, np.floor(np.exp(u))).astype(np.int64)


def grid(n: int) -> np.ndarray:
    return np.arange(n, dtype=np.float64) / n


def cfg0_signal(i: int = 0, t: int = 0, noise: float = 0.01, n: int = 1024) -> np.ndarray:
    """sin(2pi 2x) + 0.5 sin(2pi 16x) + 0.25 sin(2pi 64x) + noise*N(0,1)."""
    x = grid(n)
    s = np.sin(TWO_PI * 2 * x) + 0.5 * np.sin(TWO_PI * 16 * x) + 0.25 * np.sin(TWO_PI * 64 * x)
    if noise:
        s = s + noise * _rng(0, i, t).standard_normal(n)
    return s


def tones_signal(n: int, cfg: int, i: int, t: int = 0, kmin=2, kmax=6, fmax=None, sigma=0.05, ntones=None):
    """Sum of K integer-frequency tones (f log-uniform in [1, fmax]), A~U(0.1,1), phi~U(0,2pi), + sigma N(0,1)."""
    rng = _rng(cfg, i, t)
    K = int(ntones) if ntones is not None else int(rng.integers(kmin, kmax + 1))
    f = _loguniform_int(rng, 1, fmax if fmax is not None else n // 8, K)
    A = rng.uniform(0.1, 1.0, K)
    phi = rng.uniform(0.0, TWO_PI, K)
    x = grid(n)
    s = np.zeros(n)
    for kk in range(K):
        s += A[kk] * np.sin(TWO_PI * f[kk] * x + phi[kk])
    return s + sigma * rng.standard_normal(n)


def cfg1_signal(i: int, t: int = 0, n: int = 4096) -> np.ndarray:
    return tones_signal(n, 1, i, t)


def cfg2_signal(i: int, t: int = 0, n: int = 65536) -> np.ndarray:
    """3 AM-FM components: (1+0.5 sin(2pi fa x)) cos(2pi(f0 x + beta sin(2pi fm x)/(2pi fm))) + 0.02 N(0,1)."""
    rng = _rng(2, i, t)
    x = grid(n)
    s = np.zeros(n)
    for _ in range(3):
        fa = int(rng.integers(1, 9))
        f0 = int(_loguniform_int(rng, 4, n // 16))
        fm = int(rng.integers(1, 5))
        beta = rng.uniform(0.1, 0.4) * f0
        s += (1.0 + 0.5 * np.sin(TWO_PI * fa * x)) * np.cos(TWO_PI * (f0 * x + beta * np.sin(TWO_PI * fm * x) / (TWO_PI * fm)))
    return s + 0.02 * rng.standard_normal(n)


def cfg3_signal(i: int = 0, t: int = 0, n: int = 1 << 26) -> np.ndarray:
    return tones_signal(n, 3, i, t, fmax=1 << 20, ntones=8)


def cfg4_signal(n: int, i: int, t: int = 0) -> np.ndarray:
    """fp32 sweep signal (cfg1 recipe, f up to n/8), returned already rounded to fp32."""
    return tones_signal(n, 4 * 1000003 + n, i, t).astype(np.float32)


def make_batch(cfg: str, batch: int | None = None, n: int | None = None, start: int = 0, dtype=None) -> np.ndarray:
    """Batch [B, n] of config `cfg` signals start..start+B-1 (host, contiguous)."""
    if cfg == "cfg4":
        assert n is not None
        B = cfg4_batch(n) if batch is None else batch
        out = np.empty((B, n), dtype=np.float32)
        for b in range(B):
            out[b] = cfg4_signal(n, start + b)
        return out
    c = CONFIGS[cfg]
    n = c["n"] if n is None else n
    B = c["batch"] if batch is None else batch
    out = np.empty((B, n), dtype=np.float64 if dtype is None else dtype)
    for b in range(B):
        i = start + b
        if cfg == "cfg0":
            out[b] = cfg0_signal(i, n=n)
        elif cfg == "cfg1":
            out[b] = cfg1_signal(i, n=n)
        elif cfg == "cfg2":
            out[b] = cfg2_signal(i, n=n)
        else:
            out[b] = cfg3_signal(i, n=n)
    return out
