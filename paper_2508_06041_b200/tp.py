"""Tensor-parallel decode: one process per GPU, rows of every
linear layer split into N contiguous shards, one all-gather per op group.

Layout. Rank r holds rows [r*R', (r+1)*R') of each layer, where R' =
ceil(rows / N). The last shard is zero-padded to R' rows (zero codes, lo = hi
= 0, so the padded outputs are exactly 0), which lets every all-gather use
equal, contiguous chunks. The input vector x is replicated on all ranks.

Selector. G is replicated: option (a) of §8e. Every rank evaluates ||G x||
(or slope*||x|| + b) on the same replicated input, using the same kernel and
arithmetic, so all ranks take the same decision without an extra collective.
Exact estimators (||(W_h - W_l) x|| over all rows) would need an all-reduce
of per-shard partial norms; they and track_exact are rejected.

Data path per layer. One dpq_select_gemv launch (selector + bitplane GEMV
reading planes 0..b-1 of the local shard, runtime.py:184-193 + quant.py:95)
writes the local y shard. Then an all-gather (NCCL through torch.distributed
on GPUs; gloo with host staging in the CPU-side tests) assembles y. q/k/v
share one all-gather, and so do up/gate. The per-step glue (RMSNorm, RoPE,
attention with KV append, SiLU*up, residual adds, lm_head) restates
runtime.py:345-372 in float32 on the device. Attention runs replicated: heads
are not split, so the KV cache is per rank.

This is the straightforward NCCL baseline of §8e. The fused path (GEMV
epilogue pushing shards into peers over NVLink, with flag waits in the next
prologue) is not built yet.
"""

from __future__ import annotations

import ctypes as C
import math

import numpy as np

from . import _lib
from . import estimator as E
from . import model as M
from . import quant as Q
from .runtime import DecodeTrace, PrecisionPlan, ProvenanceError, StepRecord, DevicePlan


# ---------------------------------------------------------------------------
# sharding (host)
# ---------------------------------------------------------------------------

def shard_rows(rows: int, world: int, rank: int) -> tuple:
    """(r0, r1, rows_per_shard): contiguous row range of `rank`, padded size."""
    per = -(-rows // world)
    r0 = min(rank * per, rows)
    r1 = min(r0 + per, rows)
    return r0, r1, per


def shard_layer(q: Q.QuantizedLayer, world: int, rank: int) -> Q.QuantizedLayer:
    """Rows [r0, r1) of layer q, zero-padded to the common shard size."""
    rows, cols = q.shape
    r0, r1, per = shard_rows(rows, world, rank)
    codes = np.zeros((per, cols), dtype=np.uint16)
    lo = np.zeros(per, dtype=np.float32)
    hi = np.zeros(per, dtype=np.float32)
    codes[: r1 - r0] = q.codes[r0:r1]
    lo[: r1 - r0] = q.lo[r0:r1]
    hi[: r1 - r0] = q.hi[r0:r1]
    return Q.QuantizedLayer(codes, q.n_bits, q.b_min, lo, hi)


def gather_rows(chunks, rows: int):
    """Inverse of the sharding: concatenated padded shards -> the first `rows`."""
    return chunks.reshape(-1)[:rows] if hasattr(chunks, "reshape") else chunks[:rows]


def all_gather_flat(shard, group=None):
    """All-gather equal-size 1-D shards into (world * n,), rank order.
    NCCL gathers device tensors in place; gloo needs host tensors."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    if world == 1:
        return shard
    if dist.get_backend(group) == "nccl":
        out = torch.empty(world * shard.numel(), dtype=shard.dtype, device=shard.device)
        dist.all_gather_into_tensor(out, shard.contiguous(), group=group)
        return out
    host = shard.detach().cpu().contiguous()
    parts = [torch.empty_like(host) for _ in range(world)]
    dist.all_gather(parts, host, group=group)
    return torch.cat(parts).to(shard.device)


# ---------------------------------------------------------------------------
# engine
# ---------------------------------------------------------------------------

class TPDecodeEngine:
    """DecodeEngine (runtime.py:245-390) with tensor-parallel linears.

    Same constructor arguments as runtime.DecodeEngine plus ``group`` (a
    torch.distributed process group, default WORLD) and ``shard_store`` (a
    DeviceStore already holding this rank's padded row shards in canonical
    layer order, e.g. from synth.random_device_model(shard=...); otherwise the
    host codes of ``store`` are sharded here). ``step`` returns the float64
    logits on every rank; ``trace`` records the (identical) decisions.
    """

    def __init__(self, weights: M.ModelWeights, store: Q.BitPlaneStore, plan: PrecisionPlan,
                 store_hash: str | None = None, track_exact: bool = False,
                 async_rule: str = "prev_step", prime_from_prefill: bool = True,
                 g_dtype: str = "f16", group=None, shard_store=None):
        import torch
        import torch.distributed as dist
        if store_hash is not None and plan.store_hash and store_hash != plan.store_hash:
            raise ProvenanceError(f"plan was built against store {plan.store_hash[:12]}, "
                                  f"got {store_hash[:12]}")
        if store.config_hash != weights.config.hash():
            raise ProvenanceError("store/model config mismatch")
        if async_rule not in ("prev_step", "prev_block"):
            raise ValueError(f"unknown async rule {async_rule!r}")
        if track_exact:
            raise NotImplementedError("track_exact under tensor parallelism needs a partial-norm all-reduce")
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.weights, self.store, self.plan = weights, store, plan
        self.cfg = cfg = weights.config
        self.async_rule = async_rule
        self.prime_from_prefill = prime_from_prefill
        self.total_params = plan.total_params()
        self._ids = store.ordered_ids()
        self._index = {lid: i for i, lid in enumerate(self._ids)}
        for lid in self._ids:
            pl = plan.layers[lid]
            if pl.estimator is not None and not math.isinf(pl.T) and E.kind_code(pl.estimator) == E.EST_EXACT:
                raise NotImplementedError(f"{lid.name}: exact estimator under tensor parallelism")
        self.device = _lib.torch_device()
        # local shards: one device store + plan over the shard layers
        self._rows = [store.layers[lid].shape[0] for lid in self._ids]
        self._per = [shard_rows(r, self.world, self.rank)[2] for r in self._rows]
        if shard_store is not None:
            if [s[0] for s in shard_store.shapes] != self._per:
                raise ValueError("shard_store does not match the row sharding")
            self.dstore = shard_store
        else:
            shards = [shard_layer(store.layers[lid], self.world, self.rank) for lid in self._ids]
            self.dstore = Q.DeviceStore(shards, self.device)
        self.dplan = DevicePlan(self.dstore, [plan.layers[lid] for lid in self._ids], g_dtype)
        self._M = np.array([plan.M[l] for l in self._ids], dtype=np.float64)
        self._ops_per_step = 0
        for lid in self._ids:
            pl = plan.layers[lid]
            if not math.isinf(pl.T):
                self._ops_per_step += pl.estimator.kind.op_cost(store.layers[lid].shape[1])
        f32 = dict(device=self.device, dtype=torch.float32)
        self._embed = torch.as_tensor(np.asarray(weights.embed, dtype=np.float32), **f32)
        self._lm = torch.as_tensor(np.asarray(weights.lm_head, dtype=np.float32), **f32)
        cos, sin = M.rope_tables(cfg.seq_cap, cfg.head_dim)
        self._cos = None if cos is None else torch.as_tensor(cos, **f32)
        self._sin = None if sin is None else torch.as_tensor(sin, **f32)
        self._bit = torch.zeros(len(self._ids), dtype=torch.int32, device=self.device)
        self._est = torch.zeros(len(self._ids), dtype=torch.float32, device=self.device)
        self.reset()

    def reset(self):
        import torch
        cfg = self.cfg
        shape = (cfg.n_blocks, cfg.seq_cap, cfg.kv_heads, cfg.head_dim)
        self._k = torch.zeros(shape, dtype=torch.float32, device=self.device)
        self._v = torch.zeros(shape, dtype=torch.float32, device=self.device)
        self._pos = 0
        self._prev_inputs = {}
        self._cur_inputs = {}
        self.trace = DecodeTrace()

    @property
    def position(self) -> int:
        return self._pos

    # -- helpers (runtime.py:288-309, 383-384) ----------------------------
    def _norm(self, x):
        return x / (x.square().mean() + self.cfg.norm_eps).sqrt()

    def _rope(self, v, t):
        if self._cos is None:
            return v
        half = self._cos.shape[1]
        c, s = self._cos[t], self._sin[t]
        out = v.clone()
        v1, v2 = v[:, :half], v[:, half:2 * half]
        out[:, :half] = v1 * c - v2 * s
        out[:, half:2 * half] = v1 * s + v2 * c
        return out

    def _estimator_input(self, lid, x):
        pl = self.plan.layers[lid]
        est = pl.estimator
        if est is None or est.input_source == E.IMMEDIATE:
            return None
        if self.async_rule == "prev_block":
            prev = self._cur_inputs.get(M.LayerId(lid.block - 1, lid.kind))
        else:
            prev = self._prev_inputs.get(lid)
        return prev

    def _shard(self, lid, x, dynamic):
        """Local y shard of layer lid (selector + GEMV on the device)."""
        import torch
        i = self._index[lid]
        y = torch.empty(self._per[i], dtype=torch.float32, device=self.device)
        pl = self.plan.layers[lid]
        if not dynamic:
            _lib.call("dpq_gemv", self.dstore.handle, i, int(pl.prefill_bit), C.c_void_p(x.data_ptr()),
                      C.c_void_p(y.data_ptr()), _lib.stream_ptr())
        else:
            ein = self._estimator_input(lid, x)
            _lib.call("dpq_select_gemv", self.dplan.handle, i, C.c_void_p(x.data_ptr()),
                      C.c_void_p(ein.data_ptr()) if ein is not None else None, C.c_void_p(y.data_ptr()),
                      C.c_void_p(self._bit.data_ptr() + 4 * i), C.c_void_p(self._est.data_ptr() + 4 * i),
                      None, _lib.stream_ptr())
        self._cur_inputs[lid] = x
        return y

    def _linears(self, lids, x, dynamic):
        """y of each layer in lids (same input x): local shards, one all-gather."""
        import torch
        shards = [self._shard(lid, x, dynamic) for lid in lids]
        full = all_gather_flat(torch.cat(shards), self.group)
        tot = sum(self._per[self._index[l]] for l in lids)
        full = full.view(self.world, tot)
        out, off = [], 0
        for lid in lids:
            i = self._index[lid]
            out.append(full[:, off:off + self._per[i]].reshape(-1)[: self._rows[i]])
            off += self._per[i]
        return out

    # -- step (runtime.py:330-381) ----------------------------------------
    def step(self, token: int, dynamic: bool = True):
        import torch
        cfg = self.cfg
        t = self._pos
        if t >= cfg.seq_cap:
            raise ValueError("sequence cap exceeded")
        H, KV, hd = cfg.n_heads, cfg.kv_heads, cfg.head_dim
        qh = H // KV
        scale = 1.0 / math.sqrt(hd)
        self._cur_inputs = {}
        x = self._embed[int(token)].clone()
        for b in range(cfg.n_blocks):
            L = lambda kind: M.LayerId(b, kind)  # noqa: E731
            n1 = self._norm(x)
            q, k, v = self._linears([L("q"), L("k"), L("v")], n1, dynamic)
            q = self._rope(q.view(H, hd), t)
            k = self._rope(k.view(KV, hd), t)
            self._k[b, t] = k
            self._v[b, t] = v.view(KV, hd)
            K = self._k[b, : t + 1].repeat_interleave(qh, dim=1)      # (t+1, H, hd)
            V = self._v[b, : t + 1].repeat_interleave(qh, dim=1)
            scores = torch.einsum("hd,shd->hs", q, K) * scale
            probs = torch.softmax(scores, dim=1)
            attn = torch.einsum("hs,shd->hd", probs, V).reshape(-1).contiguous()
            (o,) = self._linears([L("o")], attn, dynamic)
            x = x + o
            n2 = self._norm(x)
            up, gate = self._linears([L("up"), L("gate")], n2, dynamic)
            h = (up * (gate / (1.0 + torch.exp(-gate)))).contiguous()
            (down,) = self._linears([L("down")], h, dynamic)
            x = x + down
        logits = self._lm @ self._norm(x)
        self._pos += 1
        if dynamic:
            bits = self._bit.cpu().numpy().astype(np.int64)
            est = self._est.cpu().numpy()
            rec = StepRecord(t, {}, {}, {}, 0.0)
            for i, lid in enumerate(self._ids):
                rec.bits[lid] = int(bits[i])
                pl = self.plan.layers[lid]
                rec.estimates[lid] = None if (math.isinf(pl.T) or np.isnan(est[i])) else float(est[i])
            rec.effective_bits = float((bits * self._M).sum() / self.total_params)
            self.trace.steps.append(rec)
            self.trace.estimator_ops += self._ops_per_step
        if dynamic or self.prime_from_prefill:
            self._prev_inputs = self._cur_inputs
        return logits.double().cpu().numpy()

    def prefill(self, tokens):
        logits = None
        for tok in tokens:
            logits = self.step(int(tok), dynamic=False)
        return logits


def decode(weights, store, plan, prompt, n_new, store_hash=None, group=None, **engine_kw):
    """Greedy decode (runtime.py:393-409) under tensor parallelism."""
    if len(prompt) == 0:
        raise ValueError("empty prompt")
    if len(prompt) + n_new > weights.config.seq_cap:
        raise ValueError("sequence cap exceeded")
    eng = TPDecodeEngine(weights, store, plan, store_hash, group=group, **engine_kw)
    logits = eng.prefill(prompt)
    out = []
    for _ in range(n_new):
        tok = int(np.argmax(logits))
        out.append(tok)
        logits = eng.step(tok, dynamic=True)
    return out, eng.trace
