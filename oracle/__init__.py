"""oracle -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.

Plain, slow, obviously-correct CPU implementations of what the FIF hot path
computes (arXiv 1802.01359, PAPER.md), used only by tests/, by
__graft_entry__.smoke() and by bench.py's cpu_baseline / --impl reference legs.
The product path (paper_1802_01359_b200) never imports this package and shares
no code with it.

  fif_oracle.c   -- time-domain DIF oracle: literally iterates s <- s - w(*)s
                    (PAPER.md:385-417), fp64, OpenMP across signals.
  direct_form.py -- CPU-DF: the paper's FFT direct form with a linear N scan
                    (PAPER.md:686-692), numpy fp64, used where TD is too slow.

Parity pins: tests/test_oracle_pins.py.  Unpinned parts are listed in DESIGN.md.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liboracle.so")
SRC_PATH = os.path.join(_HERE, "fif_oracle.c")

WINDOW_TRI_SQ = 0
WINDOW_TRI_SQ_WIDE = 1


def build(force: bool = False) -> str:
    """Compile the C oracle (plain -O2, no fast-math, no FP contraction: reading A8)."""
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(SRC_PATH):
        cmd = ["gcc", "-O2", "-std=c11", "-fopenmp", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
               SRC_PATH, "-o", LIB_PATH + ".tmp", "-lm"]
        subprocess.check_call(cmd)
        os.replace(LIB_PATH + ".tmp", LIB_PATH)
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(LIB_PATH)
        dp = ctypes.POINTER(ctypes.c_double)
        ip = ctypes.POINTER(ctypes.c_int32)
        i64, i32, d = ctypes.c_int64, ctypes.c_int32, ctypes.c_double
        L.oracle_count_extrema.argtypes = [dp, i64, d, dp]
        L.oracle_count_extrema.restype = i64
        L.oracle_filter_half_length.argtypes = [d, i64, i64, ctypes.c_int]
        L.oracle_filter_half_length.restype = i64
        L.oracle_triangle.argtypes = [i64, dp]
        L.oracle_triangle.restype = i64
        L.oracle_window.argtypes = [i64, dp]
        L.oracle_window.restype = i64
        L.oracle_inner.argtypes = [dp, i64, i64, d, i32, dp, dp, ctypes.c_int]
        L.oracle_inner.restype = i32
        L.oracle_decompose_batch.argtypes = [dp, i64, i64, ctypes.c_int, d, d, i32, i32, dp, ip, ip, ip, ip, dp,
                                             ctypes.c_int, ctypes.c_int, d]
        L.oracle_extrema_decision_margin.argtypes = [dp, i64, i64, d, d, d, d, ctypes.c_int, ctypes.c_int]
        L.oracle_extrema_decision_margin.restype = d
        L.oracle_spectral_peak.argtypes = [dp, i64, dp]
        L.oracle_spectral_peak.restype = i64
        L.oracle_inner_n0.argtypes = [dp, i64, i64, d, i32, dp, dp, ctypes.c_int]
        L.oracle_inner_n0.restype = i32
        L.oracle_dft_inf.argtypes = [dp, i64]
        L.oracle_dft_inf.restype = d
        L.oracle_decompose_batch.restype = None
        L.oracle_n0_bound.argtypes = [d]
        L.oracle_n0_bound.restype = i64
        L.oracle_num_threads.argtypes = []
        L.oracle_num_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def _dp(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _ip(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))


def count_extrema(r, scale=0.0):
    """(k, margin): k interior extrema (reading A4); margin = min nonzero |diff| / scale (max|r| if scale <= 0)."""
    r = np.ascontiguousarray(r, dtype=np.float64)
    m = np.zeros(1)
    k = lib().oracle_count_extrema(_dp(r), r.shape[0], float(scale), _dp(m))
    return int(k), float(m[0])


def filter_half_length(xi, n, k, window=WINDOW_TRI_SQ):
    return int(lib().oracle_filter_half_length(float(xi), int(n), int(k), int(window)))


def triangle(L):
    """h (unit-sum sampled triangle) as a centred array of length 2L-1 (h[j + L-1] = h_j)."""
    h = np.zeros(2 * L - 1)
    lib().oracle_triangle(int(L), _dp(h))
    return h


def window(L):
    """w = h(*)h as a centred array of length 4L-3 (w[d + 2L-2] = w_d)."""
    w = np.zeros(4 * L - 3)
    lib().oracle_window(int(L), _dp(w))
    return w


def inner(r, L, delta, max_inner, parallel=False):
    """(I-W)^N r with N chosen by the SD rule; returns (imf, N, SD_N, SD_{N-1})."""
    r = np.ascontiguousarray(r, dtype=np.float64)
    imf = np.zeros_like(r)
    sd = np.zeros(4)
    N = lib().oracle_inner(_dp(r), r.shape[0], int(L), float(delta), int(max_inner), _dp(imf), _dp(sd),
                           1 if parallel else 0)
    return imf, int(N), float(sd[0]), float(sd[1])


STOP_SD, STOP_N0 = 0, 1
MASK_EXTREMA, MASK_SPECTRAL = 0, 1


def spectral_peak(r):
    """(f*, margin): the highest-frequency significant local maximum of |DFT(r)|^2 (A20)."""
    r = np.ascontiguousarray(r, dtype=np.float64)
    m = np.zeros(1)
    f = lib().oracle_spectral_peak(_dp(r), r.shape[0], _dp(m))
    return int(f), float(m[0])


def dft_inf(r):
    """||U^T r||_inf, U the unitary DFT (reading A16), by the O(n^2) definition."""
    r = np.ascontiguousarray(r, dtype=np.float64)
    return float(lib().oracle_dft_inf(_dp(r), r.shape[0]))


def inner_n0(r, L, delta, max_inner, parallel=False):
    """A-priori rule: (I-W)^N r with N = min(N0, max_inner); returns (imf, N)."""
    r = np.ascontiguousarray(r, dtype=np.float64)
    imf = np.zeros_like(r)
    sd = np.zeros(4)
    N = lib().oracle_inner_n0(_dp(r), r.shape[0], int(L), float(delta), int(max_inner), _dp(imf), _dp(sd),
                              1 if parallel else 0)
    return imf, int(N)


def extrema_decision_margin(r, k, em, scale, tau, xi=1.6, window=WINDOW_TRI_SQ, mask=MASK_EXTREMA):
    """Reading A21: +inf if the a2/a3 decision on r is robust to the f fragile differences (|diff| <= tau*scale,
    k uncertain by +-2f), else em."""
    r = np.ascontiguousarray(r, dtype=np.float64)
    return float(lib().oracle_extrema_decision_margin(_dp(r), r.shape[0], int(k), float(em), float(scale),
                                                      float(tau), float(xi), int(window), int(mask)))


def decompose(signals, xi=1.6, delta=1e-3, max_inner=200, max_imfs=10, window=WINDOW_TRI_SQ, stop=STOP_SD,
              mask=MASK_EXTREMA, tau=1e-11):
    """Time-domain oracle decomposition of a batch [B, n] (or one signal [n]).
    stop = STOP_SD: the relative SD rule (reading A5); STOP_N0: the a-priori N0 of Thm DIF_conv_stop with
    the absolute delta (readings A16-A18).

    Returns dict: imfs [B, max_imfs+1, n], count [B], l [B, max_imfs], N [B, max_imfs],
    k [B, max_imfs+1] (extrema count at each outer step), margins [B, max_imfs+1, 2]
    (reading A21, DESIGN.md -- per outer step m: the margin of the a2/a3 decision at its head (+inf for
    the first, taken on s itself, and for decisions robust to the differences below tau * max|s|, else
    min |diff| / max|s|), and the SD margin |SD - delta| * ||iterate|| / (2 ||s||) of IMF m (the remainder
    perturbation, in units of ||s||, that can flip it); NaN where no decision was taken)."""
    s = np.ascontiguousarray(np.atleast_2d(np.asarray(signals, dtype=np.float64)))
    B, n = s.shape
    imfs = np.zeros((B, max_imfs + 1, n))
    count = np.zeros(B, dtype=np.int32)
    l = np.zeros((B, max_imfs), dtype=np.int32)
    N = np.zeros((B, max_imfs), dtype=np.int32)
    k = np.zeros((B, max_imfs + 1), dtype=np.int32)
    margins = np.zeros((B, max_imfs + 1, 2))
    lib().oracle_decompose_batch(_dp(s), B, n, int(window), float(xi), float(delta), int(max_inner), int(max_imfs),
                                 _dp(imfs), _ip(count), _ip(l), _ip(N), _ip(k), _dp(margins), int(stop), int(mask),
                                 float(tau))
    return {"imfs": imfs, "count": count, "l": l, "N": N, "k": k, "margins": margins}


def n0_bound(rhs):
    """Minimum N0 with N0^N0/(N0+1)^(N0+1) < rhs."""
    return int(lib().oracle_n0_bound(float(rhs)))


def num_threads():
    return int(lib().oracle_num_threads())
