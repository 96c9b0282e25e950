"""Tensor-parallel decode on the persistent engine (north star (4); SURVEY
§8e): the reference's per-layer matvecs (runtime.py:348-369) sharded by
output rows over N ranks, one rank per GPU (or N ranks on one device).

Layout. Rank r holds rows [r R/N, (r+1) R/N) of every linear layer: its
H/N query heads and KV/N kv heads of q/k/v (attention is head-local, the KV
cache too), d/N rows of o and down, d_ff/N rows of up and gate. The input of
every op is the full vector, replicated.

Exchange (no NCCL on the data path). Each rank's engine (dpq_engine.cu)
publishes what other ranks read into every rank's exchange arena, tile by
tile, from the epilogue that produces it: the o / up|gate / down output rows
(the row-shard all-gather, fused), the attention chunk states of its heads
(o's input windows span all heads), its estimator partials and its stage
arrivals. Arenas of other processes are mapped with CUDA IPC
(``dpq_session_tp_ipc_handle`` / ``dpq_tp_ipc_open``, peer access over
NVLink); ranks in one process on one device share pointers directly.

Selector: option (b) of §8e. G is sharded by k: rank r holds rows
[r k/N, (r+1) k/N) of each layer's projection and adds its G.x partials into
every rank's estimator set, so every rank sees the full ||G x|| and takes the
same decision (estimator.py:49-60, runtime.py:184-193) without a collective.
Linear estimators need only sum x^2, which every rank has.
"""

from __future__ import annotations

import ctypes as C
import math

import numpy as np

from . import _lib
from . import estimator as E
from . import model as M
from . import quant as Q
from .runtime import DecodeEngine, DecodeTrace, DevicePlan, PlanLayer, PrecisionPlan, ProvenanceError

IPC_HANDLE_BYTES = 64


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


def all_gather_flat(shard, group=None):
    """All-gather equal-size 1-D shards into (world * n,), rank order (host
    staging for gloo). Test and tooling helper; the engine's data path
    exchanges through peer memory."""
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


def check_shardable(cfg: M.ModelConfig, world: int):
    """Row shards must be whole heads and whole 32-row tiles."""
    kv = cfg.kv_heads
    hd = cfg.d_model // cfg.n_heads
    if world < 1 or world > 8:
        raise ValueError("tensor parallelism over 1..8 ranks")
    if cfg.n_heads % world or kv % world or cfg.d_ff % world:
        raise ValueError(f"heads {cfg.n_heads}, kv heads {kv} and d_ff {cfg.d_ff} must divide by {world}")
    for rows in (cfg.d_model // world, kv * hd // world, cfg.d_ff // world):
        if rows % 32:
            raise ValueError(f"a {world}-way shard of {rows} rows is not a whole number of 32-row tiles")


def fx_bits_of(G: np.ndarray) -> int:
    """The engine's fixed-point fraction bits for a projection G (the rule of
    dpq_plan_create), from the FULL layer's G, so every rank's shard uses the
    same scale."""
    maxl1 = float(np.max(np.sum(np.abs(G), axis=1))) if G.size else 0.0
    fb = 46 - int(math.ceil(math.log2(max(maxl1, 1e-30) * 65536.0)))
    return min(52, max(-16, fb))


def shard_plan_layers(plan: PrecisionPlan, ids, world: int, rank: int):
    """Per layer: the PlanLayer with this rank's rows [r k/N, (r+1) k/N) of the
    projection (option (b)), and the full layer's fixed-point bits."""
    out, fx = [], []
    for lid in ids:
        pl = plan.layers[lid]
        est = pl.estimator
        if est is not None and not math.isinf(pl.T) and isinstance(est.kind, E.ExactEstimator):
            raise NotImplementedError("exact estimators under tensor parallelism: the engine keeps the "
                                      "||y_h - y_l|| sets per rank (no partial-norm exchange)")
        if est is not None and hasattr(est.kind, "G") and not math.isinf(pl.T):
            G = np.ascontiguousarray(est.kind.G, dtype=np.float64)
            k = G.shape[0]
            if k % world:
                raise ValueError(f"{lid.name}: projection rank k={k} does not shard over {world} ranks")
            kl = k // world
            sub = E.ErrorEstimator(E.ProjectionEstimator(G[rank * kl:(rank + 1) * kl], kl, est.kind.seed),
                                   est.input_source, est.pair)
            out.append(PlanLayer(pl.layer, pl.prefill_bit, pl.p, pl.pair, pl.T, pl.r, sub))
            fx.append(fx_bits_of(G))
        else:
            out.append(pl)
            fx.append(None)
    return out, fx


def shard_store(store: Q.BitPlaneStore, world: int, rank: int, device=None) -> Q.DeviceStore:
    """This rank's row shards of every layer (canonical order) on the device."""
    return Q.DeviceStore([shard_layer(store.layers[lid], world, rank) for lid in store.ordered_ids()], device)


# ---------------------------------------------------------------------------
# one rank's engine
# ---------------------------------------------------------------------------

class TPDecodeEngine(DecodeEngine):
    """DecodeEngine (runtime.py:245-390) of tensor-parallel rank ``rank`` of
    ``world`` on the persistent engine. Same constructor arguments as
    runtime.DecodeEngine plus ``rank`` / ``world`` (default: the
    torch.distributed group's), ``group``, ``shard_store`` (a DeviceStore of
    this rank's row shards in canonical order; else sharded here from the
    host codes of ``store``) and ``grid`` (CTAs of this rank's engine, 0 =
    every SM). ``connect`` must run on every rank before the first step;
    ``TPDecodeEngine.create`` does it through torch.distributed (CUDA IPC
    handles exchanged with all_gather_object). Every rank returns the same
    logits and records the same decisions."""

    def __init__(self, weights: M.ModelWeights, store: Q.BitPlaneStore, plan: PrecisionPlan,
                 store_hash: str | None = None, track_exact: bool = False,
                 async_rule: str = "prev_step", prime_from_prefill: bool = True,
                 g_dtype: str = "f32", rank: int = 0, world: int = 1, shard_store_=None, grid: int = 0):
        if store_hash is not None and plan.store_hash and store_hash != plan.store_hash:
            raise ProvenanceError(f"plan was built against store {plan.store_hash[:12]}, "
                                  f"got {store_hash[:12]}")
        if store.config_hash != weights.config.hash():
            raise ProvenanceError("store/model config mismatch")
        if track_exact:
            raise NotImplementedError("track_exact under tensor parallelism: the engine keeps the "
                                      "||y_h - y_l|| sets per rank (no partial-norm exchange)")
        if async_rule not in ("prev_step", "prev_block"):
            raise ValueError(f"unknown async rule {async_rule!r}")
        cfg = weights.config
        check_shardable(cfg, world)
        self.rank, self.world = rank, world
        self.weights, self.store, self.plan = weights, store, plan
        self.cfg = cfg
        self.track_exact = False
        self.async_rule = async_rule
        self.prime_from_prefill = prime_from_prefill
        self.total_params = plan.total_params()
        self._ids = store.ordered_ids()
        self._M = np.array([plan.M[l] for l in self._ids], dtype=np.float64)
        pls = [plan.layers[l] for l in self._ids]
        self._ops_per_step = 0
        for lid, pl in zip(self._ids, pls):
            if not math.isinf(pl.T):
                self._ops_per_step += pl.estimator.kind.op_cost(store.layers[lid].shape[1])
        self._dual = [False] * len(pls)
        self._sentinel = [math.isinf(pl.T) for pl in pls]
        ds = shard_store_ if shard_store_ is not None else shard_store(store, world, rank)
        layers, fx = shard_plan_layers(plan, self._ids, world, rank)
        self.dplan = DevicePlan(ds, layers, g_dtype, fx_bits=fx)
        md = _lib.ModelDesc()
        md.n_blocks, md.d_model, md.n_heads = cfg.n_blocks, cfg.d_model, cfg.n_heads
        md.n_kv_heads, md.d_ff, md.vocab, md.seq_cap = cfg.kv_heads, cfg.d_ff, cfg.vocab, cfg.seq_cap
        md.norm_eps = cfg.norm_eps
        emb = np.ascontiguousarray(weights.embed, dtype=np.float32)
        lm = np.ascontiguousarray(weights.lm_head, dtype=np.float32)
        md.embed, md.lm_head = emb.ctypes.data, lm.ctypes.data
        md.track_exact = 0
        md.async_prev_block = int(async_rule == "prev_block")
        md.prime_from_prefill = int(prime_from_prefill)
        md.use_graph, md.use_pdl, md.use_persistent = 1, 1, 1
        td = _lib.TpDesc(rank, world, int(grid), 0)
        h = C.c_void_p()
        import torch
        from .quant import _destroy
        import weakref
        with torch.cuda.device(ds.device):
            _lib.call("dpq_session_create_tp", ds.handle, self.dplan.handle, C.byref(md), C.byref(td), C.byref(h))
        self._h = h
        self._fin = weakref.finalize(self, _destroy, "dpq_session_destroy", h.value)
        self._logits = np.empty(cfg.vocab, dtype=np.float32)
        self._opened = []
        self.reset()

    # -- peers --
    def arena(self) -> int:
        base, n = C.c_void_p(), C.c_int64()
        _lib.call("dpq_session_tp_arena", self._h, C.byref(base), C.byref(n))
        return base.value

    def ipc_handle(self) -> bytes:
        buf = (C.c_char * IPC_HANDLE_BYTES)()
        _lib.call("dpq_session_tp_ipc_handle", self._h, buf)
        return bytes(buf)

    def connect(self, peer_bases):
        """peer_bases[q]: rank q's arena in this process (own arena at rank)."""
        arr = (C.c_void_p * self.world)(*[C.c_void_p(b) for b in peer_bases])
        _lib.call("dpq_session_tp_connect", self._h, arr)

    def connect_ipc(self, handles):
        """Map the other ranks' arenas from their IPC handles (rank order)."""
        dev = self.dplan.store.device.index
        bases = []
        for q, hb in enumerate(handles):
            if q == self.rank:
                bases.append(self.arena())
                continue
            base = C.c_void_p()
            buf = C.create_string_buffer(bytes(hb), IPC_HANDLE_BYTES)
            _lib.call("dpq_tp_ipc_open", dev, buf, C.byref(base))
            self._opened.append(base.value)
            bases.append(base.value)
        self.connect(bases)

    @classmethod
    def create(cls, weights, store, plan, group=None, **kw):
        """One rank per process: rank / world from torch.distributed, IPC
        handles exchanged with all_gather_object, arenas mapped, barrier."""
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        eng = cls(weights, store, plan, rank=rank, world=world, **kw)
        handles = [None] * world
        dist.all_gather_object(handles, eng.ipc_handle(), group=group)
        eng.connect_ipc(handles)
        dist.barrier(group)
        return eng

    def close(self):
        dev = self.dplan.store.device.index
        for b in self._opened:
            try:
                _lib.call("dpq_tp_ipc_close", dev, C.c_void_p(b))
            except Exception:
                pass
        self._opened = []
        self._fin()

    # -- stepping: launch (no wait) / finish --
    def launch_step(self, token: int, dynamic: bool = True, forced_bits=None):
        if self._pos >= self.cfg.seq_cap:
            raise ValueError("sequence cap exceeded")
        fb = self._forced(forced_bits)
        _lib.call("dpq_session_step", self._h, int(token), int(bool(dynamic)),
                  C.c_void_p(fb.ctypes.data) if fb is not None else None, None)
        if dynamic:
            self._dyn_pos.append(self._pos)
            self._trace.estimator_ops += self._ops_per_step
        self._pos += 1

    def finish_step(self, want_logits: bool = True):
        if want_logits:
            _lib.call("dpq_session_logits", self._h, C.c_void_p(self._logits.ctypes.data))
            return self._logits.astype(np.float64)
        _lib.call("dpq_session_sync", self._h)
        return None

    def step(self, token: int, dynamic: bool = True, forced_bits=None, want_logits: bool = True):
        self.launch_step(token, dynamic, forced_bits)
        return self.finish_step(want_logits)

    def launch_greedy(self, n_new: int):
        if self._pos + n_new > self.cfg.seq_cap:
            raise ValueError("sequence cap exceeded")
        _lib.call("dpq_session_launch_steps", self._h, int(n_new), None)
        self.note_device_steps(n_new)

    def decode_greedy(self, n_new: int) -> list:
        if self._pos + n_new > self.cfg.seq_cap:
            raise ValueError("sequence cap exceeded")
        toks = np.zeros(max(n_new, 1), dtype=np.int32)
        _lib.call("dpq_session_decode", self._h, int(n_new), C.c_void_p(toks.ctypes.data))
        self.note_device_steps(n_new)
        return [int(t) for t in toks[:n_new]]


def decode(weights, store, plan, prompt, n_new, store_hash=None, group=None, **engine_kw):
    """Greedy decode (runtime.py:393-409) on this rank of the process group;
    every rank returns the same (tokens, DecodeTrace)."""
    if len(prompt) == 0:
        raise ValueError("empty prompt")
    eng = TPDecodeEngine.create(weights, store, plan, group=group, store_hash=store_hash, **engine_kw)
    if len(prompt) + n_new > weights.config.seq_cap:
        raise ValueError("sequence cap exceeded")
    eng.prefill(prompt)
    out = eng.decode_greedy(n_new) if n_new > 0 else []
    return out, eng.trace


# ---------------------------------------------------------------------------
# N ranks in one process on one device (tests, single-GPU demonstration)
# ---------------------------------------------------------------------------

class LocalTPGroup:
    """``world`` TP ranks of the same model in this process on the current
    device, each engine on n_sm / world CTAs, arenas shared by pointer; the
    ranks' kernels run concurrently on their own streams. Rank 0's logits,
    tokens and trace are returned; ``check_identical`` compares every rank's
    logits (they must be equal: same decisions, same reductions)."""

    def __init__(self, weights, store, plan, world: int, g_dtype: str = "f32", grid: int | None = None, **kw):
        n_sm = C.c_int()
        cc0, cc1 = C.c_int(), C.c_int()
        import torch
        _lib.call("dpq_device_info", torch.cuda.current_device(), C.byref(n_sm), C.byref(cc0), C.byref(cc1))
        g = grid if grid is not None else n_sm.value // world
        self.ranks = [TPDecodeEngine(weights, store, plan, g_dtype=g_dtype, rank=r, world=world, grid=g, **kw)
                      for r in range(world)]
        bases = [e.arena() for e in self.ranks]
        for e in self.ranks:
            e.connect(bases)
        self.world = world

    @property
    def trace(self) -> DecodeTrace:
        return self.ranks[0].trace

    def step(self, token: int, dynamic: bool = True, forced_bits=None, all_logits: bool = False):
        for e in self.ranks:
            e.launch_step(token, dynamic, forced_bits)
        lg = [e.finish_step(True) for e in self.ranks]
        return lg if all_logits else lg[0]

    def prefill(self, tokens):
        out = None
        for t in tokens:
            out = self.step(int(t), dynamic=False)
        return out

    def decode_greedy(self, n_new: int) -> list:
        for e in self.ranks[1:]:
            e.launch_greedy(n_new)
        toks = self.ranks[0].decode_greedy(n_new)
        for e in self.ranks[1:]:
            _lib.call("dpq_session_sync", e._h)
        return toks

    def close(self):
        for e in self.ranks:
            e.close()
