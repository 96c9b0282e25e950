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
# GPU: TP decode engine, two ranks on one device
# ---------------------------------------------------------------------------

def _model_and_plan():
    from test_gpu_runtime import calibrate_T, synthetic_projection_plan
    cfg = M.ModelConfig(n_blocks=2, d_model=128, n_heads=4, d_ff=352, vocab=256, seq_cap=64, n_kv_heads=2)
    w = M.init_model(3, cfg)
    store = Q.quantize_model(w, 5, 3)
    plan = synthetic_projection_plan(store, {l: (3, 4) for l in store.layers}, k=32, seed=6)
    toks = np.random.default_rng(8).integers(0, 256, 20)
    calibrate_T(w, store, plan, toks[:8])
    return w, store, plan, toks


def _tp_decode_worker(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist
    _init(rank, world, port)
    torch.cuda.set_device(0)
    w, store, plan, toks = _model_and_plan()
    eng = TP.TPDecodeEngine(w, store, plan)
    lg = [eng.step(int(toks[0]), dynamic=False)]
    for t in toks[1:]:
        lg.append(eng.step(int(t), dynamic=True))
    if rank == 0:
        ids = store.ordered_ids()
        bits = np.array([[s.bits[l] for l in ids] for s in eng.trace.steps])
        np.save(os.path.join(out_dir, f"tp{world}.npy"), {"logits": np.array(lg), "bits": bits},
                allow_pickle=True)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
def test_tp2_matches_tp1_and_engine():
    import torch.multiprocessing as mp
    from paper_2508_06041_b200 import runtime as R
    with tempfile.TemporaryDirectory() as d:
        for world in (1, 2):
            mp.spawn(_tp_decode_worker, args=(world, _free_port(), d), nprocs=world, join=True)
        r1 = np.load(os.path.join(d, "tp1.npy"), allow_pickle=True).item()
        r2 = np.load(os.path.join(d, "tp2.npy"), allow_pickle=True).item()
    # TP=2 vs TP=1: identical decisions (replicated selector), logits within fp32 tolerance
    np.testing.assert_array_equal(r2["bits"], r1["bits"])
    scale = np.max(np.abs(r1["logits"]))
    assert np.max(np.abs(r2["logits"] - r1["logits"])) <= 1e-5 * scale
    # and the persistent engine under forced-bits replay of the TP decisions
    w, store, plan, toks = _model_and_plan()
    eng = R.DecodeEngine(w, store, plan)
    lg = [eng.step(int(toks[0]), dynamic=False)]
    for t, bits in zip(toks[1:], r1["bits"]):
        lg.append(eng.step(int(t), dynamic=True, forced_bits=bits.astype(np.int8)))
    assert np.max(np.abs(np.array(lg) - r1["logits"])) <= 1e-4 * scale
