"""Host precompute of the small dense operators and the per-device C-ABI
context that carries them to the kernels.

Everything here is O(L^3) host math done once per (sensitivity, basis,
config), exactly where the reference builds the same matrices:
  Tikhonov ridge inverse        unmix.py:53-74
  Beer-Lambert fit matrix       bayes.py:99-104
  shape-prior normal matrix     bayes.py:114-129 (incl. the cond(N) > 1e13 check)
The kernels additionally need G = N^-1 C^T, which turns the shape-prior
solve N^-1 (C^T y + P e) into e + G (y - C e).
"""

from __future__ import annotations

import ctypes
import hashlib
import threading
from dataclasses import dataclass

import numpy as np
import scipy.linalg

from . import _native
from .errors import ArgumentError, IllConditionedPriorError

COND_LIMIT = 1e13  # bayes.py:33
# fp32 map path: pixels whose smallest reconstructed band is below this are
# recomputed in fp64 (profiles/r01_fallback_threshold_study.txt: fp32 error
# <= 2e-6 THb rel / 1.2e-6 SO2 abs for bands >= 1e-3, fails below 1e-4)
DEFAULT_FALLBACK_BELOW = 2e-3


def second_difference(count: int) -> np.ndarray:
    """(count - 2) x count unit-spaced [1, -2, 1] operator (bayes.py:84-93)."""
    if count < 3:
        raise ArgumentError(f"second difference needs >= 3 samples, got {count}")
    d2 = np.zeros((count - 2, count))
    rows = np.arange(count - 2)
    for shift, coef in enumerate((1.0, -2.0, 1.0)):
        d2[rows, rows + shift] = coef
    return d2


def ridge_inverse(c: np.ndarray, gamma: float) -> np.ndarray:
    """L x 3 matrix (C^T C + gamma I)^-1 C^T via the 3 x 3 push-through form."""
    return np.linalg.solve(c @ c.T + gamma * np.eye(3), c).T


def fit_matrix(xi: np.ndarray) -> np.ndarray:
    """3 x L least-squares fit matrix (xi^T xi)^-1 xi^T."""
    return np.linalg.solve(xi.T @ xi, xi.T)


@dataclass(frozen=True)
class ShapePrior:
    """P = beta D2^T D2, N = C^T C + P (Cholesky), G = N^-1 C^T."""

    prior: np.ndarray
    cho: tuple
    gain: np.ndarray

    @classmethod
    def build(cls, c: np.ndarray, beta: float) -> "ShapePrior":
        d2 = second_difference(c.shape[1])
        prior = beta * (d2.T @ d2)
        normal = c.T @ c + prior
        cond = np.linalg.cond(normal)
        if not np.isfinite(cond) or cond > COND_LIMIT:
            raise IllConditionedPriorError(
                f"shape-prior normal matrix is numerically singular (condition estimate {cond:.3e})"
            )
        cho = scipy.linalg.cho_factor(normal)
        gain = scipy.linalg.cho_solve(cho, c.T)
        return cls(prior=prior, cho=cho, gain=gain)


@dataclass(frozen=True)
class OperatorSet:
    """Everything one oxm_ctx carries (all float64, C-order)."""

    n_bands: int
    solve: np.ndarray  # L x 3
    fit_mat: np.ndarray  # 3 x L
    xi: np.ndarray  # L x 3
    sens: np.ndarray  # 3 x L
    gain: np.ndarray  # L x 3
    epsilon: float = 1e-6
    rel_tol: float = 1e-4
    max_iters: int = 20
    fallback_below: float = DEFAULT_FALLBACK_BELOW

    def key(self) -> bytes:
        h = hashlib.sha1()
        for a in (self.solve, self.fit_mat, self.xi, self.sens, self.gain):
            h.update(np.ascontiguousarray(a, dtype=np.float64).tobytes())
        h.update(repr((self.n_bands, self.epsilon, self.rel_tol, self.max_iters, self.fallback_below)).encode())
        return h.digest()


def make_operator_set(
    *,
    n_bands: int,
    solve: np.ndarray | None = None,
    xi: np.ndarray | None = None,
    sens: np.ndarray | None = None,
    gain: np.ndarray | None = None,
    epsilon: float = 1e-6,
    rel_tol: float = 1e-4,
    max_iters: int = 20,
    fallback_below: float = DEFAULT_FALLBACK_BELOW,
) -> OperatorSet:
    """Operator set with unused members zero-filled (e.g. a fit-only context)."""
    L = int(n_bands)
    if not 3 <= L <= _native.MAX_BANDS:
        raise ArgumentError(f"the CUDA kernels support 3..{_native.MAX_BANDS} bands, got {L}")
    z3 = np.zeros((L, 3))
    unit = np.column_stack([np.zeros((L, 2)), np.ones(L)])  # placeholder basis: (0, 0, 1) rows
    xi_ = unit if xi is None else np.asarray(xi, dtype=np.float64)
    fit = np.zeros((3, L)) if xi is None else fit_matrix(xi_)
    return OperatorSet(
        n_bands=L,
        solve=z3 if solve is None else np.asarray(solve, dtype=np.float64),
        fit_mat=fit,
        xi=xi_,
        sens=np.zeros((3, L)) if sens is None else np.asarray(sens, dtype=np.float64),
        gain=z3 if gain is None else np.asarray(gain, dtype=np.float64),
        epsilon=float(epsilon),
        rel_tol=float(rel_tol),
        max_iters=int(max_iters),
        fallback_below=float(fallback_below),
    )


class DeviceContext:
    """Owns one oxm_ctx (host-side struct; operators travel as kernel params)."""

    def __init__(self, ops: OperatorSet, device_index: int):
        lib = _native.load()
        self._keep = [np.ascontiguousarray(a, dtype=np.float64) for a in (ops.solve, ops.fit_mat, ops.xi, ops.sens, ops.gain)]
        s, f, x, c, g = self._keep
        st = _native.Operators(
            n_bands=ops.n_bands,
            max_iters=ops.max_iters,
            epsilon=ops.epsilon,
            rel_tol=ops.rel_tol,
            fallback_below=ops.fallback_below,
            solve=s.ctypes.data,
            fit_mat=f.ctypes.data,
            xi=x.ctypes.data,
            sens=c.ctypes.data,
            gain=g.ctypes.data,
        )
        handle = ctypes.c_void_p()
        _native.check(lib.oxm_ctx_create(device_index, ctypes.byref(st), ctypes.byref(handle)), "oxm_ctx_create")
        self.handle = handle.value
        self.ops = ops
        self.device_index = device_index
        self._lib = lib

    def __del__(self):
        h, self.handle = getattr(self, "handle", None), None
        if h:
            try:
                self._lib.oxm_ctx_destroy(h)
            except Exception:
                pass


_ctx_lock = threading.Lock()
_ctx_cache: dict[tuple[bytes, int], DeviceContext] = {}


def context(ops: OperatorSet, device_index: int) -> DeviceContext:
    key = (ops.key(), int(device_index))
    with _ctx_lock:
        ctx = _ctx_cache.get(key)
        if ctx is None:
            if len(_ctx_cache) > 256:
                _ctx_cache.clear()
            ctx = DeviceContext(ops, int(device_index))
            _ctx_cache[key] = ctx
        return ctx
