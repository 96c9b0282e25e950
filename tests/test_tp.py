"""Tensor parallelism: row sharding, shard all-gather and the
TP decode engine.

Multi-process with the gloo backend (world size 2): the CPU test checks the
sharding and gather against the oracle; the GPU test runs two ranks on
cuda:0 (gloo stages the shards through host memory) and compares TP=2 with
TP=1 and with the persistent engine: same decisions, logits within the fp32
tolerance (SURVEY §8c / §8e parity rule).
"""

import os
import socket
import tempfile

import numpy as np
import pytest

from oracle import dpq_oracle as O
from paper_2508_06041_b200 import model as M
from paper_2508_06041_b200 import quant as Q
from paper_2508_06041_b200 import tp as TP


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _init(rank, world, port):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


def test_shard_rows_cover_and_pad():
    for rows in (1, 31, 32, 33, 4096, 14336):
        for world in (1, 2, 4, 8):
            got = []
            for r in range(world):
                r0, r1, per = TP.shard_rows(rows, world, r)
                assert 0 <= r1 - r0 <= per and per * world >= rows
                got.extend(range(r0, r1))
            assert got == list(range(rows))


def _gather_worker(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist
    _init(rank, world, port)
    rng = np.random.default_rng(5)
    res = {}
    for rows, cols in ((33, 40), (64, 32), (7, 16)):
        W = rng.standard_normal((rows, cols)).astype(np.float32) / np.sqrt(cols)
        q = O.quantize_layer(W, 5, 3)
        layer = Q.QuantizedLayer(q.codes, q.n_bits, q.b_min, q.lo, q.hi)
        x = rng.standard_normal(cols)
        sh = TP.shard_layer(layer, world, rank)
        y_shard = O.dequantize(sh, 4) @ x                      # oracle on the shard (checker)
        full = TP.all_gather_flat(torch.as_tensor(y_shard), None)
        res[f"{rows}x{cols}"] = (full.numpy()[:rows], O.dequantize(layer, 4) @ x)
    if rank == 0:
        np.save(os.path.join(out_dir, "gather.npy"), res, allow_pickle=True)
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_gemv_gathers_to_full_layer_gloo2():
    import torch.multiprocessing as mp
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_gather_worker, args=(2, _free_port(), d), nprocs=2, join=True)
        res = np.load(os.path.join(d, "gather.npy"), allow_pickle=True).item()
    for name, (got, ref) in res.items():
        np.testing.assert_allclose(got, ref, rtol=0, atol=1e-12, err_msg=name)


# ---------------------------------------------------------------------------
# GPU: the TP engine (row shards, peer-memory exchange), ranks on one device
# ---------------------------------------------------------------------------

def _model_and_plan(g_seed=6):
    from test_gpu_runtime import calibrate_T, synthetic_projection_plan
    cfg = M.ModelConfig(n_blocks=2, d_model=256, n_heads=4, d_ff=512, vocab=256, seq_cap=64, n_kv_heads=2)
    w = M.init_model(3, cfg)
    store = Q.quantize_model(w, 5, 3)
    plan = synthetic_projection_plan(store, {l: (3, 4) for l in store.layers}, k=32, seed=g_seed)
    toks = np.random.default_rng(8).integers(0, 256, 20)
    calibrate_T(w, store, plan, toks[:8])
    return w, store, plan, toks


def test_check_shardable():
    cfg = M.ModelConfig(n_blocks=1, d_model=4096, n_heads=32, d_ff=14336, n_kv_heads=8)
    for world in (1, 2, 4, 8):
        TP.check_shardable(cfg, world)
    with pytest.raises(ValueError):
        TP.check_shardable(M.ModelConfig(n_blocks=1, d_model=256, n_heads=4, d_ff=352, n_kv_heads=2), 2)


def test_plan_shards_G_by_k():
    """Option (b): rank r gets rows [r k/N, (r+1) k/N) of each projection; the
    fixed-point scale is the full layer's on every rank."""
    from test_gpu_runtime import synthetic_projection_plan
    cfg = M.ModelConfig(n_blocks=1, d_model=64, n_heads=2, d_ff=128, vocab=32, seq_cap=8)
    w = M.init_model(0, cfg)
    store = Q.quantize_model(w, 5, 3)
    plan = synthetic_projection_plan(store, {l: (3, 4) for l in store.layers}, k=32, seed=1)
    ids = store.ordered_ids()
    for world in (2, 4):
        parts = [TP.shard_plan_layers(plan, ids, world, r) for r in range(world)]
        for i, lid in enumerate(ids):
            G = plan.layers[lid].estimator.kind.G
            got = np.concatenate([p[0][i].estimator.kind.G for p in parts])
            np.testing.assert_array_equal(got, G)
            assert {p[1][i] for p in parts} == {TP.fx_bits_of(G)}


@pytest.mark.gpu
@pytest.mark.parametrize("g_dtype", ["f32", "f16"])
def test_tp2_engine_matches_tp1_and_oracle(g_dtype):
    """Two ranks (one process, one device, 74 CTAs each): identical decisions
    and logits to the TP=1 engine (the same per-(tile, window) partials and
    fixed-point sums), every rank the same logits, and the oracle under
    forced replay of the decisions within the fp32 tolerance."""
    from paper_2508_06041_b200 import _lib
    from paper_2508_06041_b200 import runtime as R
    w, store, plan, toks = _model_and_plan()
    ids = store.ordered_ids()
    grp = TP.LocalTPGroup(w, store, plan, 2, g_dtype=g_dtype)
    assert all(_lib.load().dpq_session_is_persistent(e._h) == 2 for e in grp.ranks)
    lg2 = [grp.step(int(toks[0]), dynamic=False, all_logits=True)]
    for t in toks[1:]:
        lg2.append(grp.step(int(t), dynamic=True, all_logits=True))
    lg2 = np.array(lg2)                                     # [step][rank][vocab]
    np.testing.assert_array_equal(lg2[:, 0], lg2[:, 1])
    bits2 = np.array([[s.bits[l] for l in ids] for s in grp.trace.steps])
    bits2b = np.array([[s.bits[l] for l in ids] for s in grp.ranks[1].trace.steps])
    np.testing.assert_array_equal(bits2, bits2b)
    highs = np.mean(bits2 == 4)
    assert 0.1 < highs < 0.9
    eng = R.DecodeEngine(w, store, plan, g_dtype=g_dtype)
    lg1 = [eng.step(int(toks[0]), dynamic=False)] + [eng.step(int(t)) for t in toks[1:]]
    bits1 = np.array([[s.bits[l] for l in ids] for s in eng.trace.steps])
    np.testing.assert_array_equal(bits2, bits1)
    scale = np.max(np.abs(lg1))
    assert np.max(np.abs(lg2[:, 0] - np.array(lg1))) <= 1e-6 * scale
    est1 = np.array([[s.estimates[l] for l in ids] for s in eng.trace.steps])
    est2 = np.array([[s.estimates[l] for l in ids] for s in grp.trace.steps])
    np.testing.assert_array_equal(est1, est2)
    # oracle, replaying the decisions
    eo = O.Engine(w, store.layers, plan.layers, plan.M)
    eo.forced = [{O.key(l): int(b) for l, b in zip(ids, row)} for row in bits2]
    ref = [eo.step(int(toks[0]), dynamic=False)] + [eo.step(int(t)) for t in toks[1:]]
    assert np.max(np.abs(lg2[:, 0] - np.array(ref))) <= 2e-5 * np.max(np.abs(ref))
    grp.close()
    eng.close()


@pytest.mark.gpu
def test_tp2_device_greedy_loop():
    """dpq_session_decode on both ranks (argmax fed back on the device, one
    launch per rank): the TP=1 engine's tokens and decisions."""
    from paper_2508_06041_b200 import runtime as R
    w, store, plan, toks = _model_and_plan()
    grp = TP.LocalTPGroup(w, store, plan, 2)
    grp.prefill(toks[:5])
    out2 = grp.decode_greedy(12)
    out1, tr1 = R.decode(w, store, plan, toks[:5], 12, g_dtype="f32")
    assert out2 == out1
    ids = store.ordered_ids()
    assert [[s.bits[l] for l in ids] for s in grp.trace.steps] == [[s.bits[l] for l in ids] for s in tr1.steps]
    grp.close()


@pytest.mark.gpu
def test_tp_rejects_exact_sets():
    """track_exact (and exact estimators) keep their ||y_h - y_l|| sets per
    rank, so a tensor-parallel session with them is refused with the reason
    instead of running with partial norms (host check in tp.py; the C-ABI
    session refuses them too)."""
    w, store, plan, _ = _model_and_plan()
    with pytest.raises(NotImplementedError, match="tensor parallelism"):
        TP.LocalTPGroup(w, store, plan, 2, track_exact=True)
