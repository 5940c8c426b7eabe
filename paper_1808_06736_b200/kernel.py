"""ES kernel parameters and host-side kernel math (mirrors esnufft.kernel).

phi_beta(z) = exp(beta (sqrt(1 - z^2) - 1)) on |z| <= 1, 0 outside.  The
parameter recipe, Gauss-Legendre rule, phi-hat corrections and the
piecewise-polynomial fit are computed by the C++ runtime of
libesnufft_b200.so (esn_math.cpp) -- the same code the GPU plans use -- and
exposed here with the reference's names and error behaviour
(esnufft/kernel.py:51-412).
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass
from functools import lru_cache

import numpy as np

from . import _lib
from .errors import BadToleranceError, SizeError

MIN_WIDTH = 2
MAX_WIDTH = 16
MIN_TOLERANCE = 1e-15
MAX_TOLERANCE = 1e-1
SUPPORTED_SIGMAS = (2.0, 1.25)
GAMMA_SAFETY = 0.976
EPS64 = float(np.finfo(np.float64).eps)


@dataclass(frozen=True)
class KernelParams:
    """w (2..16), beta, sigma (2.0 / 1.25), gamma, p_quad (kernel.py:51-84)."""

    w: int
    beta: float
    sigma: float
    gamma: float
    p_quad: int

    def __post_init__(self):
        if not (MIN_WIDTH <= self.w <= MAX_WIDTH):
            raise BadToleranceError(f"kernel width {self.w} outside [{MIN_WIDTH}, {MAX_WIDTH}]")
        if not self.beta > 0:
            raise BadToleranceError(f"beta must be positive, got {self.beta}")
        if self.sigma not in SUPPORTED_SIGMAS:
            raise BadToleranceError(
                f"sigma {self.sigma} unsupported; choose one of {SUPPORTED_SIGMAS}")
        if not 0.0 < self.gamma <= 1.0:
            raise BadToleranceError(f"safety factor gamma {self.gamma:.6f} outside (0, 1]")
        if self.p_quad < math.ceil(1.5 * self.w + 2):
            raise BadToleranceError(
                f"p_quad {self.p_quad} below ceil(1.5 w + 2) = {math.ceil(1.5 * self.w + 2)}")

    def to_c(self) -> _lib.KernelParamsC:
        return _lib.KernelParamsC(self.w, self.beta, self.sigma, self.gamma, self.p_quad)


def _from_c(kp: _lib.KernelParamsC) -> KernelParams:
    return KernelParams(w=int(kp.w), beta=float(kp.beta), sigma=float(kp.sigma),
                        gamma=float(kp.gamma), p_quad=int(kp.p_quad))


def params_for_width(w: int, sigma: float = 2.0) -> KernelParams:
    kp = _lib.KernelParamsC()
    _lib.check(_lib.lib.esn_params_for_width(int(w), float(sigma), ctypes.byref(kp)))
    return _from_c(kp)


def select_params(tolerance: float, sigma: float = 2.0) -> KernelParams:
    kp = _lib.KernelParamsC()
    tolerance = float(tolerance)
    if math.isnan(tolerance):
        raise BadToleranceError("tolerance nan outside supported range")
    _lib.check(_lib.lib.esn_select_params(tolerance, float(sigma), ctypes.byref(kp)))
    return _from_c(kp)


def class_tolerance(w: int, sigma: float = 2.0) -> float:
    return float(_lib.lib.esn_class_tolerance(int(w), float(sigma)))


def es_eval(z, beta: float):
    """phi_beta at real arguments, exactly zero outside [-1, 1]."""
    z = np.asarray(z, dtype=np.float64)
    scalar = z.ndim == 0
    z = np.atleast_1d(z)
    out = np.zeros_like(z)
    inside = np.abs(z) <= 1.0
    out[inside] = np.exp(beta * (np.sqrt(1.0 - z[inside] ** 2) - 1.0))
    return float(out[0]) if scalar else out


@lru_cache(maxsize=64)
def gauss_legendre(n: int) -> tuple[np.ndarray, np.ndarray]:
    if n < 1:
        raise SizeError(f"gauss_legendre needs n >= 1, got {n}")
    x = np.empty(n)
    w = np.empty(n)
    _lib.check(_lib.lib.esn_gauss_legendre(int(n), x.ctypes.data_as(_lib.P_dbl),
                                           w.ctypes.data_as(_lib.P_dbl)))
    x.setflags(write=False)
    w.setflags(write=False)
    return x, w


def kernel_ft(params: KernelParams, alpha: float, ks) -> np.ndarray:
    """psi-hat(k) = 2 alpha sum_j w_j phi(q_j) cos(alpha k q_j)."""
    if alpha <= 0:
        raise SizeError(f"alpha must be positive, got {alpha}")
    ks = np.ascontiguousarray(np.atleast_1d(np.asarray(ks, dtype=np.float64)))
    out = np.empty(ks.shape)
    kp = params.to_c()
    _lib.check(_lib.lib.esn_kernel_ft(ctypes.byref(kp), float(alpha), ks.size,
                                      ks.ctypes.data_as(_lib.P_dbl), out.ctypes.data_as(_lib.P_dbl)))
    return out


def fseries_correction(params: KernelParams, n: int, num_modes: int) -> np.ndarray:
    """p_k = h / psi-hat(k), centered ascending k, by phase winding."""
    if num_modes < 1 or n < num_modes:
        raise SizeError(f"need 1 <= num_modes <= n, got num_modes={num_modes}, n={n}")
    out = np.empty(int(num_modes))
    kp = params.to_c()
    _lib.check(_lib.lib.esn_fseries_correction(ctypes.byref(kp), int(n), int(num_modes),
                                               out.ctypes.data_as(_lib.P_dbl)))
    return out


@dataclass(frozen=True)
class PiecewisePoly:
    """w pieces of degree w+3, coeffs (w, w+4) highest degree first."""

    w: int
    degree: int
    coeffs: np.ndarray
    beta: float
    fit_residual: float


@lru_cache(maxsize=64)
def _poly_cached(w: int, beta: float, sigma: float, gamma: float, p_quad: int) -> PiecewisePoly:
    kp = _lib.KernelParamsC(w, beta, sigma, gamma, p_quad)
    coeffs = np.empty((w, w + 4))
    res = ctypes.c_double(0.0)
    _lib.check(_lib.lib.esn_piecewise_poly(ctypes.byref(kp), coeffs.ctypes.data_as(_lib.P_dbl),
                                           ctypes.byref(res)))
    coeffs.setflags(write=False)
    return PiecewisePoly(w=w, degree=w + 3, coeffs=coeffs, beta=beta, fit_residual=float(res.value))


def build_piecewise_poly(params: KernelParams) -> PiecewisePoly:
    return _poly_cached(params.w, params.beta, params.sigma, params.gamma, params.p_quad)


def _row_t(w: int, x_frac: float) -> float:
    if w % 2 == 0:
        return 1.0 - 2.0 * x_frac
    return -2.0 * x_frac if x_frac < 0.5 else 2.0 - 2.0 * x_frac


def poly_eval_row(poly: PiecewisePoly, x_frac: float) -> np.ndarray:
    """Kernel values at the w ordinates of a point with fractional offset
    x_frac in [0, 1) (kernel.py:378-397)."""
    if not 0.0 <= x_frac < 1.0:
        raise SizeError(f"x_frac must lie in [0, 1), got {x_frac}")
    t = _row_t(poly.w, x_frac)
    row = poly.coeffs[:, 0].copy()
    for q in range(1, poly.degree + 1):
        row = row * t + poly.coeffs[:, q]
    return row


def exact_eval_row(params: KernelParams, x_frac: float) -> np.ndarray:
    """Same row by direct evaluation (kernel.py:400-412)."""
    if not 0.0 <= x_frac < 1.0:
        raise SizeError(f"x_frac must lie in [0, 1), got {x_frac}")
    w = params.w
    if w % 2 == 0:
        z0 = (2.0 / w) * (1.0 - w / 2.0 - x_frac)
    elif x_frac < 0.5:
        z0 = (2.0 / w) * (-(w - 1) / 2.0 - x_frac)
    else:
        z0 = (2.0 / w) * (1.0 - (w - 1) / 2.0 - x_frac)
    return es_eval(z0 + (2.0 / w) * np.arange(w), params.beta)
