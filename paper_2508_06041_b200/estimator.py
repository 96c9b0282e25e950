"""Relative-error estimators of the precision selector (drop-in for the
runtime half of ``dpq.estimator``, /root/reference/pkg/src/dpq/estimator.py).

Types mirror the reference: ``LinearEstimator`` (estimator.py:35-46),
``ProjectionEstimator`` (:49-60), ``ExactEstimator`` (:63-73),
``ErrorEstimator`` (:76-83), input-source tags (:26-27) and
``resolve_input_source`` (:267-272). ``estimate`` runs on the GPU; inside a
decode step the same estimators are evaluated by the fused op kernel
(libdpq_b200: op_kernel P1 + decider), never here.

The offline half (calibration, the fitter) is out of scope for the hot path.
``translate_threshold`` (estimator.py:106-121, returns a ``ThresholdEntry``)
and ``build_projection`` (estimator.py:190-200, returns a
``ProjectionEstimator``) keep the reference signatures; the product
``A @ dW`` is formed on the GPU from device-dequantized planes.
"""

from __future__ import annotations

import ctypes as C
import math
import weakref
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from . import quant as Q

IMMEDIATE = "immediate"
PREVIOUS_RESIDUAL = "previous_residual"
DEFAULT_K = 64
EST_NONE, EST_LINEAR, EST_PROJECTION, EST_EXACT = 0, 1, 2, 3


def _to_device(x):
    import torch
    dev = _lib.torch_device()
    if isinstance(x, torch.Tensor):
        return x.to(device=dev, dtype=torch.float32).contiguous()
    return torch.as_tensor(np.asarray(x, dtype=np.float32), device=dev)


def exact_error(layer: Q.QuantizedLayer, l: int, h: int, x) -> float:
    """||(W_h - W_l) x|| from one device pass over planes 0..h-1 (the l-plane
    sum is a prefix of the h-plane sum; lo cancels)."""
    if l >= h:
        raise Q.QuantError(f"need l < h, got ({l}, {h})")
    ds, i = layer.device_handle()
    return ds.exact_error(i, l, h, _to_device(x))


class _DevEstimator:
    """dpq_estimator handle (linear / projection) for standalone estimate()."""

    def __init__(self, kind, cols, slope=0.0, intercept=0.0, G=None, k=0):
        sd = _lib.SelDesc()
        sd.est_kind = kind
        sd.slope, sd.intercept = float(slope), float(intercept)
        sd.k = int(k)
        self._G = None
        if G is not None:
            self._G = np.ascontiguousarray(G, dtype=np.float64)
            sd.G = self._G.ctypes.data
        h = C.c_void_p()
        dev = _lib.torch_device()
        _lib.call("dpq_estimator_create", dev.index, C.byref(sd), int(cols), C.byref(h))
        self.handle = h
        self._fin = weakref.finalize(self, Q._destroy, "dpq_estimator_destroy", h.value)

    def __call__(self, x) -> float:
        xt = _to_device(x)
        out = C.c_double()
        _lib.call("dpq_estimator_eval", self.handle, C.c_void_p(xt.data_ptr()), C.byref(out),
                  _lib.stream_ptr())
        return float(out.value)


@dataclass
class LinearEstimator:
    slope: float
    intercept: float
    r2: float
    _dev: dict = field(default_factory=dict, repr=False, compare=False)

    def estimate(self, x) -> float:
        cols = np.shape(x)[-1]
        if cols not in self._dev:
            self._dev[cols] = _DevEstimator(EST_LINEAR, cols, self.slope, self.intercept)
        return self._dev[cols](x)

    def op_cost(self, cols: int) -> int:
        return cols + 2


@dataclass
class ProjectionEstimator:
    G: np.ndarray               # (k, cols)
    k: int
    seed: int
    calibrated: bool = False
    _dev: object = field(default=None, repr=False, compare=False)

    def estimate(self, x) -> float:
        if self._dev is None:
            self._dev = _DevEstimator(EST_PROJECTION, self.G.shape[1], G=self.G, k=self.G.shape[0])
        return self._dev(x)

    def op_cost(self, cols: int) -> int:
        return self.k * cols


@dataclass
class ExactEstimator:
    layer: Q.QuantizedLayer
    l: int
    h: int

    def estimate(self, x) -> float:
        return exact_error(self.layer, self.l, self.h, x)

    def op_cost(self, cols: int) -> int:
        return self.layer.shape[0] * cols


@dataclass
class ErrorEstimator:
    kind: object                # LinearEstimator | ProjectionEstimator | ExactEstimator
    input_source: str           # IMMEDIATE or PREVIOUS_RESIDUAL
    pair: tuple                 # (l, h)

    def estimate(self, x) -> float:
        return self.kind.estimate(x)


def kind_code(est) -> int:
    if est is None:
        return EST_NONE
    k = est.kind
    if isinstance(k, LinearEstimator) or (hasattr(k, "slope") and not hasattr(k, "G")):
        return EST_LINEAR
    if isinstance(k, ProjectionEstimator) or hasattr(k, "G"):
        return EST_PROJECTION
    return EST_EXACT


def resolve_input_source(lid) -> str:
    """q/k/v/up layers past block 0 may estimate from the previous input."""
    return PREVIOUS_RESIDUAL if (lid.residual_fed and lid.block > 0) else IMMEDIATE


def empirical_quantile(sorted_vals, r: float) -> float:
    """Ceil-index quantile, index ceil(r*n)-1 clamped (estimator.py:94-103)."""
    n = len(sorted_vals)
    idx = min(max(math.ceil(r * n - 1e-9) - 1, 0), n - 1)
    return float(sorted_vals[idx])


@dataclass
class ThresholdEntry:
    """estimator.py:86-91."""
    layer: object
    T: float                    # may be +/- inf
    r_quantile: float
    pair: tuple


def translate_threshold(err_list, p: float, l: int) -> ThresholdEntry:
    """Threshold of a (l, l+1) layer from an error list (estimator.py:106-121):
    r = 1 - (p - l); r >= 1 -> +inf (always low), r <= 0 -> -inf (always
    high), else the empirical r-quantile. The list is used in the order
    given, like the reference (callers pass it sorted)."""
    err_list = np.asarray(err_list, dtype=np.float64)
    if len(err_list) == 0:
        raise ValueError("empty error list")
    if not (l <= p <= l + 1):
        raise ValueError(f"p={p} outside [{l}, {l + 1}]")
    r = 1.0 - (p - l)
    if r >= 1.0:
        T = math.inf
    elif r <= 0.0:
        T = -math.inf
    else:
        T = empirical_quantile(err_list, r)
    return ThresholdEntry(None, T, r, (l, l + 1))


def projection_matrix(delta_rows_fn, rows: int, k: int, seed: int, A=None) -> np.ndarray:
    """G = A @ dW with A ~ N(0,1)/sqrt(k) (estimator.py:196-200). ``delta_rows_fn``
    returns dW as a float64 (rows, cols) array or a CUDA tensor; the product
    is formed on the GPU for large layers."""
    if k < 1:
        raise ValueError("k must be >= 1")
    if A is None:
        A = np.random.default_rng(seed).standard_normal((k, rows)) / np.sqrt(k)
    dW = delta_rows_fn()
    import torch
    if isinstance(dW, torch.Tensor):
        At = torch.as_tensor(A, device=dW.device, dtype=dW.dtype)
        return (At @ dW).double().cpu().numpy()
    return A @ dW


def build_projection(layer: Q.QuantizedLayer, l: int, h: int, k: int, seed: int,
                     A=None) -> ProjectionEstimator:
    """estimator.py:190-200: G = A @ (W_h - W_l), A seeded N(0,1)/sqrt(k);
    dW is dequantized on the device in fp64 (quant.py:83-92)."""
    if k < 1:
        raise ValueError("k must be >= 1")
    ds, i = layer.device_handle()

    def dW():
        d = ds.dequantize(i, h)
        d -= ds.dequantize(i, l)
        return d

    return ProjectionEstimator(projection_matrix(dW, layer.shape[0], k, seed, A), k, seed)
