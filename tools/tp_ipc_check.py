"""Multi-process tensor-parallel check on ONE device (needs CUDA MPS so the
ranks' persistent kernels run concurrently): 2 processes, each a TP rank
with its own engine on n_sm / 2 CTAs, arenas exchanged through CUDA IPC
handles (torch.distributed gloo all_gather_object), greedy decode compared
with the single-GPU engine.

    nvidia-cuda-mps-control -d; python tools/tp_ipc_check.py
"""
import os
import socket
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np  # noqa: E402


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def worker(rank, world, port, out):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2508_06041_b200 import tp as TP
    from test_tp import _model_and_plan
    w, store, plan, toks = _model_and_plan()
    eng = TP.TPDecodeEngine.create(w, store, plan, grid=148 // world)
    eng.prefill(toks[:5])
    out_toks = eng.decode_greedy(12)
    ids = store.ordered_ids()
    bits = [[s.bits[l] for l in ids] for s in eng.trace.steps]
    if rank == 0:
        np.save(out, {"toks": out_toks, "bits": bits}, allow_pickle=True)
    dist.barrier()
    eng.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    import tempfile
    import torch.multiprocessing as mp
    from paper_2508_06041_b200 import runtime as R
    with tempfile.TemporaryDirectory() as d:
        out = os.path.join(d, "r.npy")
        mp.spawn(worker, args=(2, _port(), out), nprocs=2, join=True)
        got = np.load(out, allow_pickle=True).item()
    import torch
    torch.cuda.set_device(0)
    from test_tp import _model_and_plan
    w, store, plan, toks = _model_and_plan()
    ref, tr = R.decode(w, store, plan, toks[:5], 12, g_dtype="f32")
    ids = store.ordered_ids()
    ok = got["toks"] == ref and got["bits"] == [[s.bits[l] for l in ids] for s in tr.steps]
    print("tp2 over IPC (2 processes):", "OK" if ok else "MISMATCH", got["toks"], ref)
    sys.exit(0 if ok else 1)
