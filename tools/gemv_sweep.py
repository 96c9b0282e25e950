"""Single-layer any-precision GEMV + selector sweep (BASELINE config 2).

    python tools/gemv_sweep.py [--reps 20] [--out profiles/r1_gemv_sweep.jsonl]

Shapes 4096x4096, 14336x4096 and 4096x14336, an 8-bit nested store (random
codes: bandwidth does not depend on the values), batch 1:
  * static: ``dpq_gemv`` at b = 3..8, planes 0..b-1 only (quant.py:95-99);
  * dynamic: ``dpq_select_gemv`` with a k=64 projection selector (f16 G) on
    the pair (b, b+1), thresholds set so half of the layer copies decide high
    (realized b + 0.5), i.e. the fused selector prologue + GEMV
    (runtime.py:184-193).
Each launch streams a different copy of the layer (copies x planes > 126 MB
L2, so every launch reads HBM); launches are captured into one CUDA graph
(falls back to plain stream launches if capture fails) and timed with CUDA
events on the launching stream. GB/s counts algorithmic bytes:
rows*cols*b/8 + 8*rows (lo, span) + 4*cols (x) + 4*rows (y) [+ 2*k*cols G].
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2508_06041_b200 import _lib  # noqa: E402
from paper_2508_06041_b200 import estimator as E  # noqa: E402
from paper_2508_06041_b200 import model as M  # noqa: E402
from paper_2508_06041_b200 import quant as Q  # noqa: E402
from paper_2508_06041_b200 import runtime as R  # noqa: E402

SHAPES = [(4096, 4096), (14336, 4096), (4096, 14336)]
K = 64


def timed(launch, n_launch, reps):
    """ms per launch: graph of n_launch launches, replayed reps times."""
    s = torch.cuda.Stream()
    graph = None
    try:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            for i in range(n_launch):                          # warm every copy outside capture
                launch(C.c_void_p(s.cuda_stream), i, 1)        # (first use builds its program)
            torch.cuda.synchronize()
            with torch.cuda.graph(g, stream=s):
                for i in range(n_launch):
                    launch(C.c_void_p(torch.cuda.current_stream().cuda_stream), i, 0)
        graph = g
    except Exception as e:                                    # noqa: BLE001
        print("graph capture failed, plain launches:", e, file=sys.stderr)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sp = C.c_void_p(s.cuda_stream)
    with torch.cuda.stream(s):
        for _ in range(2):                                    # warm-up
            graph.replay() if graph else [launch(sp, i, 0) for i in range(n_launch)]
        torch.cuda.synchronize()
        e0.record(s)
        for _ in range(reps):
            if graph:
                graph.replay()
            else:
                for i in range(n_launch):
                    launch(sp, i, 0)
        e1.record(s)
        torch.cuda.synchronize()
    return e0.elapsed_time(e1) / (reps * n_launch), graph is not None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--out", default="")
    ap.add_argument("--quick", action="store_true", help="static 3 / 4 / 8 bits and dynamic (3, 4) only")
    ap.add_argument("--shape", default="", help="ROWSxCOLS: this shape only")
    ap.add_argument("--bits", default="", help="comma list of static bits (default 3..8)")
    ap.add_argument("--no-dynamic", action="store_true")
    ap.add_argument("--copies", type=int, default=0, help="layer copies (default: > 300 MB in total)")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    dev = torch.device("cuda:0")
    out = []
    shapes = [tuple(int(v) for v in args.shape.split("x"))] if args.shape else SHAPES
    for rows, cols in shapes:
        n_copy = args.copies or max(8, int(np.ceil(300e6 / (rows * cols * 3 / 8))))
        gen = torch.Generator(device=dev).manual_seed(rows + cols)
        specs = []
        rng = np.random.default_rng(0)
        for _ in range(n_copy):
            codes = torch.randint(0, 256, (rows, cols), dtype=torch.uint8, device=dev, generator=gen)
            lo = (-rng.random(rows) - 0.5).astype(np.float32)
            hi = (rng.random(rows) + 0.5).astype(np.float32)
            specs.append((codes, lo, hi, 8, 3))
        ds = Q.DeviceStore.from_device_codes(specs, dev)
        del specs
        torch.cuda.empty_cache()
        x = torch.randn(cols, device=dev)
        x = x / x.pow(2).mean().sqrt()
        y = torch.empty(rows, device=dev)
        base = rows * cols
        small = 8 * rows + 4 * cols + 4 * rows
        stat = {}
        sbits = [int(v) for v in args.bits.split(",")] if args.bits else ((3, 4, 8) if args.quick else range(3, 9))
        for b in sbits:
            def launch(sp, i, warm, b=b):
                _lib.call("dpq_gemv", ds.handle, i % n_copy, b, C.c_void_p(x.data_ptr()),
                          C.c_void_p(y.data_ptr()), sp)
            ms, graphed = timed(launch, n_copy, args.reps)
            gbps = (base * b / 8 + small) / (ms * 1e-3) / 1e9
            stat[b] = ms
            out.append({"shape": [rows, cols], "mode": "static", "bits": b, "us": ms * 1e3,
                        "GBps": gbps, "copies": n_copy, "graph": graphed})
            print(json.dumps(out[-1]), flush=True)
        # dynamic: projection selector, pair (b, b+1), half the copies high
        xs = x.double().cpu().numpy()
        for b in (() if args.no_dynamic else (3,) if args.quick else range(3, 8)):
            pls, n_high = [], 0
            for i in range(n_copy):
                G = np.random.default_rng(100 + i).standard_normal((K, cols)) / np.sqrt(cols)
                est = float(np.linalg.norm(G @ x.cpu().numpy().astype(np.float64)))
                T = est * (0.9 if i % 2 == 0 else 1.1)
                n_high += i % 2 == 0
                eo = E.ErrorEstimator(E.ProjectionEstimator(G, K, 0), E.IMMEDIATE, (b, b + 1))
                pls.append(R.PlanLayer(M.LayerId(i, "q"), b + 1, b + 0.5, (b, b + 1), T, 0.5, eo))
            dp = R.DevicePlan(ds, pls, "f16")
            bit = torch.zeros(1, dtype=torch.int32, device=dev)
            est_o = torch.zeros(1, device=dev)

            def launch(sp, i, warm):
                _lib.call("dpq_select_gemv", dp.handle, i % n_copy, C.c_void_p(x.data_ptr()), None,
                          C.c_void_p(y.data_ptr()), C.c_void_p(bit.data_ptr()),
                          C.c_void_p(est_o.data_ptr()), None, sp)
            ms, graphed = timed(launch, n_copy, args.reps)
            rb = b + n_high / n_copy
            t_static = stat[b] + (stat[b + 1] - stat[b]) * (rb - b)
            gbps = (base * rb / 8 + small + 2 * K * cols) / (ms * 1e-3) / 1e9
            out.append({"shape": [rows, cols], "mode": "dynamic", "pair": [b, b + 1], "realized_bits": rb,
                        "us": ms * 1e3, "GBps": gbps, "selector_overhead": ms / t_static - 1.0,
                        "copies": n_copy, "graph": graphed})
            print(json.dumps(out[-1]), flush=True)
            del dp
        del xs
        ds.close()
        torch.cuda.empty_cache()
    if args.out:
        with open(args.out, "w") as f:
            for r in out:
                f.write(json.dumps(r) + "\n")


if __name__ == "__main__":
    main()
