"""Synthetic models and plans for the large benchmark configurations
(cfg3-5 use init_model-law random weights and synthetic plans,
because the reference planner is infeasible at 7B+).

Offline tooling, not the decode hot path: weights are drawn and quantized on
the GPU (dpq_quantize_device, float64 semantics of quant.py:43-64), projection
matrices G = A dW (estimator.py:190-200) are formed from the device
dequantization, and thresholds are calibrated as per-layer quantiles of the
estimates seen on a calibration run (the r-quantile rule of
estimator.py:106-121 with r = 1 - (p - l)).
"""

from __future__ import annotations

import ctypes as C
import math

import numpy as np

from . import _lib
from . import estimator as E
from . import model as M
from . import quant as Q
from . import runtime as R


def random_device_model(cfg: M.ModelConfig, n_bits: int, b_min: int, seed: int = 0,
                        keep_host_blocks: int = 0, shard=None):
    """init_model-law weights (W ~ N(0, 1/cols)) generated and quantized on the
    GPU. Returns (ModelWeights with embed/lm_head only, DeviceBitPlaneStore,
    host_layers) where host_layers holds QuantizedLayer copies of the first
    ``keep_host_blocks`` blocks (for the CPU baseline slice).

    shard=(world, rank): also return, as a 4th value, a DeviceStore of this
    rank's row shards (tp.shard_rows, zero-padded) of every layer, quantized
    from the same weights (per-row quantization: identical codes).
    """
    import torch
    dev = _lib.torch_device()
    rng = np.random.default_rng(seed)
    d = cfg.d_model
    embed = rng.normal(0.0, 1.0, (cfg.vocab, d)).astype(np.float32)
    lm_head = (rng.normal(0.0, 1.0, (cfg.vocab, d)) * (0.1 / np.sqrt(d))).astype(np.float32)
    gen = torch.Generator(device=dev)
    gen.manual_seed(seed)
    shapes, host = {}, {}
    # streaming build: each layer is generated, quantized and repacked into the
    # store's bitplanes before the next one exists (full-depth 70B fits)
    ds = Q.DeviceStore.empty(dev)
    sds = Q.DeviceStore.empty(dev) if shard is not None else None
    for lid in M.layer_ids(cfg):
        rows, cols = M.layer_shape(cfg, lid)
        W = torch.randn((rows, cols), generator=gen, device=dev, dtype=torch.float32)
        W.mul_(1.0 / math.sqrt(cols))
        codes = torch.empty((rows, cols), dtype=torch.int16, device=dev)
        lo = torch.empty(rows, device=dev)
        hi = torch.empty(rows, device=dev)
        _lib.call("dpq_quantize_device", dev.index, C.c_void_p(W.data_ptr()), rows, cols, n_bits,
                  C.c_void_p(codes.data_ptr()), C.c_void_p(lo.data_ptr()), C.c_void_p(hi.data_ptr()),
                  _lib.stream_ptr())
        del W
        lo_h, hi_h = lo.cpu().numpy(), hi.cpu().numpy()
        if shard is not None:
            from . import tp as TP
            world, rank = shard
            r0, r1, per = TP.shard_rows(rows, world, rank)
            sc = torch.zeros((per, cols), dtype=torch.int16, device=dev)
            sc[: r1 - r0] = codes[r0:r1]
            slo = np.zeros(per, dtype=np.float32)
            shi = np.zeros(per, dtype=np.float32)
            slo[: r1 - r0] = lo_h[r0:r1]
            shi[: r1 - r0] = hi_h[r0:r1]
            sds.append(sc, slo, shi, n_bits, b_min)
            del sc
        ds.append(codes, lo_h, hi_h, n_bits, b_min)
        shapes[lid] = (rows, cols)
        if lid.block < keep_host_blocks:
            host[lid] = Q.QuantizedLayer(codes.cpu().numpy().view(np.uint16), n_bits, b_min, lo_h, hi_h)
        del codes
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    store = Q.DeviceBitPlaneStore(cfg.hash(), n_bits, b_min, shapes, ds)
    if shard is not None:
        return M.ModelWeights(cfg, embed, lm_head, {}), store, host, sds
    return M.ModelWeights(cfg, embed, lm_head, {}), store, host


def projection_plan(store, pairs: dict, prefill_bits: dict, k: int = E.DEFAULT_K, seed: int = 0,
                    method: str = "dp", target: float = float("nan"), use_async: bool = False) -> R.PrecisionPlan:
    """Projection estimator per dynamic layer, G = A (W_h - W_l), A ~ N(0,1)/sqrt(k)
    seeded per layer; thresholds start at +inf (calibrate_thresholds sets them).
    use_async: residual-fed layers past block 0 estimate from the previous
    input (estimator.py:267-272, 286; build_dp_plan(use_async=True))."""
    import torch
    ds = store.device_store()
    ids = store.ordered_ids()
    layers = {}
    for i, lid in enumerate(ids):
        l, h = pairs[lid]
        if l == h:
            layers[lid] = R.PlanLayer(lid, prefill_bits[lid], float(l), (l, l), np.inf, 1.0, None)
            continue
        rows = store.layers[lid].shape[0]
        A = torch.as_tensor(np.random.default_rng(seed + i).standard_normal((k, rows)) / np.sqrt(k),
                            device=ds.device)
        dW = ds.dequantize(i, h)
        dW -= ds.dequantize(i, l)
        G = (A @ dW).cpu().numpy()
        del dW
        src = E.resolve_input_source(lid) if use_async else E.IMMEDIATE
        est = E.ErrorEstimator(E.ProjectionEstimator(G, k, seed), src, (l, h))
        layers[lid] = R.PlanLayer(lid, prefill_bits[lid], l + 0.5, (l, h), np.inf, 0.5, est)
    torch.cuda.empty_cache()
    return R.PrecisionPlan(method, target, float("nan"), layers, store.param_counts())


def calibrate_thresholds(weights, store, plan, tokens, high_rate: dict | float = 0.5, **engine_kw):
    """Set each dynamic layer's T to the (1 - high_rate) quantile of the
    estimates recorded over one teacher-forced calibration pass (T = 1e300
    during the pass keeps every estimator running and every layer low)."""
    dyn = [lid for lid, pl in plan.layers.items() if pl.estimator is not None]
    for lid in dyn:
        plan.layers[lid].T = 1e300
    eng = R.DecodeEngine(weights, store, plan, **engine_kw)
    eng.step(int(tokens[0]), dynamic=False, want_logits=False)
    for t in tokens[1:]:
        eng.step(int(t), dynamic=True, want_logits=False)
    for lid in dyn:
        vals = np.sort([s.estimates[lid] for s in eng.trace.steps])
        r = 1.0 - (high_rate[lid] if isinstance(high_rate, dict) else high_rate)
        plan.layers[lid].T = E.empirical_quantile(vals, r)
        plan.layers[lid].r = r
    eng.close()
    return plan
