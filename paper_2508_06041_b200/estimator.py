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


# ---------------------------------------------------------------------------
# Offline calibration on the GPU: the planner's inputs at
# 7B+ widths, where the reference's numpy path (fp64 dense dequantized
# matrices, estimator.py:132-165, 208-264) does not fit a CPU. Float64
# throughout (the reference's arithmetic): layers dequantized on the device
# (dpq_dequantize, quant.py:67-80), the batch forward and the projection
# descent as fp64 device matmuls.
# ---------------------------------------------------------------------------

R2_GATE = 0.9                # estimator.py:21
CALIB_EPOCHS = 200           # estimator.py:23
CALIB_STEP = 1e-3            # estimator.py:24


@dataclass
class ErrorSamples:
    """estimator.py:124-129."""
    errors: np.ndarray          # collection order
    norms: np.ndarray           # paired ||x||
    sorted_errors: np.ndarray
    inputs: np.ndarray          # (n, cols) captured layer inputs


def _forward_inputs(weights, mat, tokens, cfg):
    """model.py:286-345 batch causal forward on the device in fp64 with the
    per-layer input capture of model.layer_inputs (model.py:466-477): n1 for
    q/k/v, the attention output for o, n2 for up/gate, h for down. GQA by
    head grouping (kv heads repeated). mat(lid) -> fp64 device (rows, cols)."""
    import torch
    from . import model as M
    dev = _lib.torch_device()
    f64 = torch.float64
    T = len(tokens)
    H, hd = cfg.n_heads, cfg.d_model // cfg.n_heads
    KV = cfg.kv_heads
    half = hd // 2
    inv = M.ROPE_BASE ** (-np.arange(half, dtype=np.float64) * 2.0 / hd)
    ang = np.arange(T, dtype=np.float64)[:, None] * inv[None, :]
    cos = torch.as_tensor(np.cos(ang), device=dev)[:, None, :]
    sin = torch.as_tensor(np.sin(ang), device=dev)[:, None, :]

    def rope(v):
        out = v.clone()
        a, b = v[..., :half], v[..., half:2 * half]
        out[..., :half] = a * cos - b * sin
        out[..., half:2 * half] = a * sin + b * cos
        return out

    def norm(x):
        return x * (1.0 / torch.sqrt(torch.mean(x * x, dim=-1, keepdim=True) + cfg.norm_eps))

    emb = torch.as_tensor(np.asarray(weights.embed, dtype=np.float32), device=dev)
    x = emb[torch.as_tensor(np.asarray(tokens, dtype=np.int64), device=dev)].to(f64)
    mask = torch.triu(torch.ones((T, T), dtype=torch.bool, device=dev), diagonal=1)
    captured = {}
    for b in range(cfg.n_blocks):
        ids = {k: M.LayerId(b, k) for k in M.KINDS}
        n1 = norm(x)
        for k in ("q", "k", "v"):
            captured[ids[k]] = n1
        q = rope((n1 @ mat(ids["q"]).T).reshape(T, H, hd))
        kk = rope((n1 @ mat(ids["k"]).T).reshape(T, KV, hd))
        v = (n1 @ mat(ids["v"]).T).reshape(T, KV, hd)
        if H // KV > 1:
            kk = kk.repeat_interleave(H // KV, dim=1)
            v = v.repeat_interleave(H // KV, dim=1)
        sc = torch.einsum("thd,shd->hts", q, kk) * (1.0 / math.sqrt(hd))
        sc = sc.masked_fill(mask[None], float("-inf"))
        sc = sc - sc.max(dim=-1, keepdim=True).values
        e = torch.exp(sc)
        pr = e / e.sum(dim=-1, keepdim=True)
        attn = torch.einsum("hts,shd->thd", pr, v).reshape(T, cfg.d_model)
        captured[ids["o"]] = attn
        x = x + attn @ mat(ids["o"]).T
        n2 = norm(x)
        captured[ids["up"]] = captured[ids["gate"]] = n2
        gate = n2 @ mat(ids["gate"]).T
        h = (n2 @ mat(ids["up"]).T) * (gate * (1.0 / (1.0 + torch.exp(-gate))))
        captured[ids["down"]] = h
        x = x + h @ mat(ids["down"]).T
    return captured


def collect_error_samples(weights, store, pairs: dict, max_bits: dict, calib) -> dict:
    """estimator.py:132-165 on the device: forward passes with every layer at
    its maximum precision B[i]; per calibration token and layer, the exact
    error ||(W_h - W_l) x|| of the layer's (l, h) pair, ||x|| and x."""
    import torch
    samples = list(calib)
    if not samples:
        raise ValueError("empty calibration set")
    ds = store.device_store()
    index = {lid: i for i, lid in enumerate(store.ordered_ids())}
    cfg = weights.config
    # max-bit matrices: dequantized once and kept while they fit the budget
    # (7-8B: all of them, 56 GB fp64), else again per calibration chunk
    budget = [64 << 30]
    cache = {}

    def mat(lid):
        if lid in cache:
            return cache[lid]
        m = ds.dequantize(index[lid], int(max_bits[lid]))
        if m.numel() * 8 <= budget[0]:
            cache[lid] = m
            budget[0] -= m.numel() * 8
        return m

    # phase 1: the forward passes, capturing every layer's inputs
    xs = {lid: [] for lid in pairs}
    for tokens in samples:
        inputs = _forward_inputs(weights, mat, tokens, cfg)
        for lid in pairs:
            xs[lid].append(inputs[lid])
    cache.clear()
    torch.cuda.empty_cache()
    # phase 2: per layer, dW = W_h - W_l (quant.py:83-92) and the exact errors
    out = {}
    for lid, (l, h) in pairs.items():
        if l >= h:
            raise Q.QuantError(f"need l < h, got ({l}, {h})")
        d = ds.dequantize(index[lid], h)
        d -= ds.dequantize(index[lid], l)
        X = torch.cat(xs[lid])
        e = torch.linalg.norm(X @ d.T, dim=1).cpu().numpy()
        out[lid] = ErrorSamples(e, torch.linalg.norm(X, dim=1).cpu().numpy(), np.sort(e), X.cpu().numpy())
        del d, X
        xs[lid] = None
    return out


def fit_linear(err_list, norm_list):
    """estimator.py:168-187: least squares error ~ slope ||x|| + intercept,
    accepted iff R^2 > 0.9; a LinearEstimator or None."""
    err = np.asarray(err_list, dtype=np.float64)
    nrm = np.asarray(norm_list, dtype=np.float64)
    if len(err) < 3:
        return None
    nbar, ebar = nrm.mean(), err.mean()
    sxx = np.sum((nrm - nbar) ** 2)
    sxy = np.sum((nrm - nbar) * (err - ebar))
    if sxx == 0:
        return None
    slope = sxy / sxx
    intercept = ebar - slope * nbar
    resid = err - (slope * nrm + intercept)
    sst = np.sum((err - ebar) ** 2)
    r2 = 1.0 - float(np.sum(resid ** 2) / sst) if sst > 0 else 1.0
    if r2 <= R2_GATE:
        return None
    return LinearEstimator(float(slope), float(intercept), r2)


def mean_relative_error(est_vals, exact_vals, floor=1e-12) -> float:
    """estimator.py:203-205."""
    exact_vals = np.maximum(np.asarray(exact_vals, dtype=np.float64), floor)
    return float(np.mean(np.abs(np.asarray(est_vals) - exact_vals) / exact_vals))


def calibrate_projection(est: ProjectionEstimator, inputs, exact_errors, epochs: int = CALIB_EPOCHS,
                         step: float = CALIB_STEP):
    """estimator.py:208-264 on the device in fp64: gradient descent on G of
    the squared relative gap between ||G x|| and the exact error; a step is
    taken only if the calibration-set mean relative error does not grow
    (halving it up to 30 times, doubling after an accepted step), five
    epochs without an acceptable step end the descent, and a final metric
    worse than the start restores G (warning). Returns (estimator, history,
    warning)."""
    import torch
    dev = _lib.torch_device()
    X = torch.as_tensor(np.asarray(inputs, dtype=np.float64), device=dev)
    e = torch.clamp(torch.as_tensor(np.asarray(exact_errors, dtype=np.float64), device=dev), min=1e-12)
    G0 = np.array(est.G, dtype=np.float64, copy=True)
    G = torch.as_tensor(G0, device=dev).clone()
    n = e.shape[0]

    def metric(Gm):
        vals = torch.linalg.norm(X @ Gm.T, dim=1)
        return float(torch.mean(torch.abs(vals - e) / e))

    cur = metric(G)
    history = [cur]
    stuck = 0
    step_cur = step
    for _ in range(epochs):
        proj = X @ G.T                                          # (n, k)
        norms = torch.clamp(torch.linalg.norm(proj, dim=1), min=1e-12)
        coef = 2.0 * (norms - e) / (e * e * norms * n)
        grad = (proj * coef[:, None]).T @ X                     # (k, cols)
        s = step_cur
        accepted = False
        for _ in range(30):
            cand = G - s * grad
            cand_m = metric(cand)
            if cand_m <= cur:
                G, cur = cand, cand_m
                accepted = True
                step_cur = s * 2.0
                break
            s *= 0.5
        history.append(cur)
        if accepted:
            stuck = 0
        else:
            stuck += 1
            if stuck >= 5:
                break
    warning = False
    Gh = G.cpu().numpy()
    if cur > history[0]:
        warning = True
        Gh = G0
    return ProjectionEstimator(Gh, est.k, est.seed, calibrated=True), history, warning
