"""The model's batch forward / backward (drop-in for ``dpq.model.forward``,
``backward``, ``teacher_forced_loss``; /root/reference/pkg/src/dpq/model.py
286-345, 363-372, 382-460) as float64 device graphs.

These serve the planner-side callers of the reference API (sensitivity
scores, calibration inputs); the decode hot path does not use them. The
forward restates model.py:286-345 (GQA by head grouping, as the engine);
backward differentiates the same graph (autograd in fp64) and returns the
reference's types: (loss, GradientBundle(weight_grads, output_grads), tape).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from . import model as M


@dataclass
class BlockTape:
    """model.py:256-274."""
    x_in: np.ndarray
    n1: np.ndarray
    inv1: np.ndarray
    q_rot: np.ndarray
    k_rot: np.ndarray
    v: np.ndarray
    probs: np.ndarray
    attn_cat: np.ndarray
    x_mid: np.ndarray
    n2: np.ndarray
    inv2: np.ndarray
    up: np.ndarray
    gate: np.ndarray
    sig: np.ndarray
    h: np.ndarray


@dataclass
class ForwardTape:
    """model.py:276-283."""
    tokens: np.ndarray
    blocks: list
    x_final: np.ndarray
    inv_f: np.ndarray
    normed_f: np.ndarray
    logits: np.ndarray
    provider_mats: dict


@dataclass
class GradientBundle:
    """model.py:374-379."""
    weight_grads: dict
    output_grads: dict


def full_precision_provider(weights: M.ModelWeights):
    return lambda lid: weights.linears[lid]


def _graph(weights, tokens, provider, grad: bool):
    """The forward on the device; returns (logits, tape parts, W / y tensors)."""
    import torch
    cfg = weights.config
    dev = _lib.torch_device()
    f64 = torch.float64
    T = len(tokens)
    if T > cfg.seq_cap:
        raise ValueError(f"sequence length {T} exceeds seq_cap {cfg.seq_cap}")
    if provider is None:
        provider = full_precision_provider(weights)
    H, hd, KV = cfg.n_heads, cfg.d_model // cfg.n_heads, cfg.kv_heads
    half = hd // 2
    inv = M.ROPE_BASE ** (-np.arange(half, dtype=np.float64) * 2.0 / hd)
    ang = np.arange(T, dtype=np.float64)[:, None] * inv[None, :]
    cos = torch.as_tensor(np.cos(ang), device=dev)[:, None, :]
    sin = torch.as_tensor(np.sin(ang), device=dev)[:, None, :]

    def rope(v):
        a, b = v[..., :half], v[..., half:2 * half]
        return torch.cat([a * cos - b * sin, a * sin + b * cos, v[..., 2 * half:]], dim=-1)

    def norm(x):
        inv_ = 1.0 / torch.sqrt(torch.mean(x * x, dim=-1, keepdim=True) + cfg.norm_eps)
        return x * inv_, inv_

    mats, Ws, ys = {}, {}, {}

    def W(lid):
        m = np.asarray(provider(lid), dtype=np.float64)
        mats[lid] = m
        w = torch.as_tensor(m, device=dev).requires_grad_(grad)
        Ws[lid] = w
        return w

    def lin(x, lid):
        y = x @ W(lid).T
        if grad:
            y.retain_grad()
        ys[lid] = y
        return y

    tok = torch.as_tensor(np.asarray(tokens, dtype=np.int64), device=dev)
    x = torch.as_tensor(np.asarray(weights.embed, dtype=np.float32), device=dev)[tok].to(f64)
    mask = torch.triu(torch.ones((T, T), dtype=torch.bool, device=dev), diagonal=1)
    blocks = []
    for b in range(cfg.n_blocks):
        ids = {k: M.LayerId(b, k) for k in M.KINDS}
        x_in = x
        n1, inv1 = norm(x)
        q = rope(lin(n1, ids["q"]).reshape(T, H, hd))
        k = rope(lin(n1, ids["k"]).reshape(T, KV, hd))
        v = lin(n1, ids["v"]).reshape(T, KV, hd)
        kk, vv = (k.repeat_interleave(H // KV, dim=1), v.repeat_interleave(H // KV, dim=1)) if H // KV > 1 else (k, v)
        sc = torch.einsum("thd,shd->hts", q, kk) * (1.0 / math.sqrt(hd))
        sc = sc.masked_fill(mask[None], float("-inf"))
        sc = sc - sc.max(dim=-1, keepdim=True).values
        e = torch.exp(sc)
        pr = e / e.sum(dim=-1, keepdim=True)
        attn = torch.einsum("hts,shd->thd", pr, vv).reshape(T, cfg.d_model)
        x_mid = x_in + lin(attn, ids["o"])
        n2, inv2 = norm(x_mid)
        up = lin(n2, ids["up"])
        gate = lin(n2, ids["gate"])
        sig = 1.0 / (1.0 + torch.exp(-gate))
        h = up * (gate * sig)
        x = x_mid + lin(h, ids["down"])
        blocks.append((x_in, n1, inv1, q, k, v, pr, attn, x_mid, n2, inv2, up, gate, sig, h))
    normed_f, inv_f = norm(x)
    logits = normed_f @ torch.as_tensor(np.asarray(weights.lm_head, dtype=np.float32), device=dev).to(f64).T
    return logits, blocks, x, inv_f, normed_f, mats, Ws, ys


def _np(t):
    return t.detach().cpu().numpy()


def _tape(tokens, blocks, x, inv_f, normed_f, logits, mats):
    return ForwardTape(np.asarray(tokens, dtype=np.int64), [BlockTape(*[_np(a) for a in bt]) for bt in blocks],
                       _np(x), _np(inv_f), _np(normed_f), _np(logits), mats)


def forward(weights: M.ModelWeights, tokens, provider=None, want_tape: bool = False):
    """model.py:286-345: logits (T, vocab) float64, and the tape if requested."""
    import torch
    tokens = np.asarray(tokens, dtype=np.int64)
    with torch.no_grad():
        logits, blocks, x, inv_f, normed_f, mats, _, _ = _graph(weights, tokens, provider, grad=False)
    lg = _np(logits)
    if not want_tape:
        return lg, None
    return lg, _tape(tokens, blocks, x, inv_f, normed_f, logits, mats)


def token_losses(logits, tokens):
    """model.py:354-360: per-position next-token cross entropy (T - 1)."""
    tokens = np.asarray(tokens, dtype=np.int64)
    z = logits[:-1]
    z = z - z.max(axis=-1, keepdims=True)
    lse = np.log(np.exp(z).sum(axis=-1))
    return lse - z[np.arange(len(tokens) - 1), tokens[1:]]


def teacher_forced_loss(weights: M.ModelWeights, tokens, provider=None):
    """model.py:363-372: (mean loss, exp(loss), per-token losses)."""
    tokens = np.asarray(tokens, dtype=np.int64)
    if len(tokens) < 2:
        raise ValueError("need at least 2 tokens")
    logits, _ = forward(weights, tokens, provider)
    per_token = token_losses(logits, tokens)
    loss = float(per_token.mean())
    return loss, float(np.exp(loss)), per_token


def backward(weights: M.ModelWeights, tokens, provider=None):
    """model.py:382-460: (loss, GradientBundle(dL/dW, dL/dy per linear layer), tape)."""
    import torch
    tokens = np.asarray(tokens, dtype=np.int64)
    T = len(tokens)
    if T < 2:
        raise ValueError("need at least 2 tokens")
    logits, blocks, x, inv_f, normed_f, mats, Ws, ys = _graph(weights, tokens, provider, grad=True)
    tgt = torch.as_tensor(tokens[1:], device=logits.device)
    loss = torch.nn.functional.cross_entropy(logits[:-1], tgt)      # mean over the T - 1 positions
    loss.backward()
    wg = {lid: _np(w.grad) for lid, w in Ws.items()}
    og = {lid: _np(y.grad) for lid, y in ys.items()}
    tape = _tape(tokens, blocks, x, inv_f, normed_f, logits, mats)
    return float(loss.item()), GradientBundle(wg, og), tape
