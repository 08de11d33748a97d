"""CPU oracle for TAG's SFB gradient-synchronisation hot path (arXiv 2302.06126).

TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline and
`--impl reference` legs may import this package. The product library (paper_2302_06126_b200/,
libtag.so) never imports, links or calls it, and the two share no code: the only thing both sides
use is the seeded input generator in paper_2302_06126_b200/synth.py, which holds none of the
method's arithmetic.

Contents
  tag_oracle.c  fp64 dense route, SFB route, per-entry sums, bias gradient (both routes),
                SGD-momentum, Adam, RNE bf16 cast (plain C)
  selector.py   exact-integer / Fraction selector, byte counts, ring-AllReduce and ILP formulas

Parity status: every function here is pinned by tests/test_oracle.py against values the paper or
SPEC print, closed forms, invariants, brute force (exact rationals) or a library routine. No
function is "parity unpinned".
"""
import ctypes
import os
import subprocess

import numpy as np

from . import selector  # noqa: F401  (re-export)

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "tag_oracle.c")
_lib = None


def build(force=False):
    """Compile tag_oracle.c with gcc (-O2, no FMA contraction, no fast-math) into liboracle.so."""
    if not force and os.path.exists(_SO) and os.path.getmtime(_SO) >= os.path.getmtime(_SRC):
        return _SO
    cmd = ["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC", "-shared",
           "-std=c11", "-o", _SO + ".tmp", _SRC, "-lm"]
    subprocess.check_call(cmd)
    os.replace(_SO + ".tmp", _SO)
    return _SO


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_SO)
        i64, p = ctypes.c_int64, ctypes.c_void_p
        for name in ("oracle_dense_sum", "oracle_dense_dw", "oracle_sfb_sum", "oracle_sfb_dw"):
            fn = getattr(lib, name)
            fn.argtypes = [i64, i64, i64, i64, p, p, p]
            fn.restype = None
        lib.oracle_sfb_sum_entries.argtypes = [i64, i64, i64, i64, p, p, i64, p, p]
        lib.oracle_sfb_sum_entries.restype = None
        lib.oracle_sgd_momentum.argtypes = [i64, p, p, p, ctypes.c_double, ctypes.c_double,
                                            ctypes.c_double]
        lib.oracle_sgd_momentum.restype = None
        lib.oracle_cast_bf16.argtypes = [i64, p, p]
        lib.oracle_cast_bf16.restype = None
        lib.oracle_adam.argtypes = [i64, p, p, p, p] + [ctypes.c_double] * 5 + [i64]
        lib.oracle_adam.restype = None
        for name in ("oracle_dense_bias_sum", "oracle_sfb_bias_sum"):
            fn = getattr(lib, name)
            fn.argtypes = [i64, i64, i64, p, p]
            fn.restype = None
        _lib = lib
    return _lib


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def _shapes(X, dY):
    n, B, M = X.shape
    n2, B2, N = dY.shape
    assert (n, B) == (n2, B2), "X is (n, B, M) and dY is (n, B, N)"
    return n, B, M, N


def _route(name, X, dY):
    X, dY = _f64(X), _f64(dY)
    n, B, M, N = _shapes(X, dY)
    out = np.empty((M, N), dtype=np.float64)
    getattr(_load(), name)(n, B, M, N, _ptr(X), _ptr(dY), _ptr(out))
    return out


def dense_sum(X, dY):
    """S = sum_r X_r^T dY_r (per-replica triple loop, rank-order sum). X: (n,B,M), dY: (n,B,N)."""
    return _route("oracle_dense_sum", X, dY)


def dense_dw(X, dY):
    """dW = S / (nB) by the dense (AllReduce) route."""
    return _route("oracle_dense_dw", X, dY)


def sfb_sum(X, dY):
    """S = sum_k X_all[k]^T (outer) dY_all[k] (rank-1 accumulation over the gathered factors)."""
    return _route("oracle_sfb_sum", X, dY)


def sfb_dw(X, dY):
    """dW = S / (nB) by the SFB route."""
    return _route("oracle_sfb_dw", X, dY)


def sfb_sum_entries(X, dY, flat_idx):
    """S[m][j] for each flat index m*N + j, computed one by one."""
    X, dY = _f64(X), _f64(dY)
    n, B, M, N = _shapes(X, dY)
    idx = np.ascontiguousarray(flat_idx, dtype=np.int64)
    out = np.empty(idx.shape[0], dtype=np.float64)
    _load().oracle_sfb_sum_entries(n, B, M, N, _ptr(X), _ptr(dY), idx.shape[0], _ptr(idx),
                                   _ptr(out))
    return out


def sgd_momentum(dW, W, v, lr, mu, wd):
    """One SGD-momentum step in fp64; returns (W', v') (inputs are not modified)."""
    dW = _f64(dW).ravel()
    W2 = _f64(W).ravel().copy()
    v2 = _f64(v).ravel().copy()
    _load().oracle_sgd_momentum(dW.size, _ptr(dW), _ptr(W2), _ptr(v2), lr, mu, wd)
    return W2.reshape(np.shape(W)), v2.reshape(np.shape(v))


def cast_bf16_bits(x):
    """RNE fp32 -> bf16; returns the uint16 bit patterns."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    out = np.empty(x.shape, dtype=np.uint16)
    _load().oracle_cast_bf16(x.size, _ptr(x), _ptr(out))
    return out


def bf16_bits_to_f64(bits):
    """Exact value of bf16 bit patterns (a bf16 is the top half of an fp32)."""
    b = np.ascontiguousarray(bits, dtype=np.uint16).astype(np.uint32) << 16
    return b.view(np.float32).astype(np.float64)


def _bias(name, dY):
    dY = _f64(dY)
    n, B, N = dY.shape
    out = np.empty(N, dtype=np.float64)
    getattr(_load(), name)(n, B, N, _ptr(dY), _ptr(out))
    return out


def dense_bias_sum(dY):
    """S_b = sum_r sum_b dY_r[b] (per-replica bias gradients, rank-order sum). dY: (n, B, N)."""
    return _bias("oracle_dense_bias_sum", dY)


def sfb_bias_sum(dY):
    """S_b = sum_k dY_all[k] (column sums of the gathered dY_all)."""
    return _bias("oracle_sfb_bias_sum", dY)


def sfb_bias(dY):
    """db = S_b / (nB) by the SFB route."""
    n, B, _ = np.shape(dY)
    return sfb_bias_sum(dY) / float(n * B)


def adam(dW, W, m, v, lr, b1, b2, eps, wd, t):
    """One Adam step (torch.optim.Adam semantics, step t >= 1) in fp64; returns (W', m', v')."""
    dW = _f64(dW).ravel()
    W2, m2, v2 = (_f64(x).ravel().copy() for x in (W, m, v))
    _load().oracle_adam(dW.size, _ptr(dW), _ptr(W2), _ptr(m2), _ptr(v2), lr, b1, b2, eps, wd, t)
    shape = np.shape(W)
    return W2.reshape(shape), m2.reshape(shape), v2.reshape(shape)
