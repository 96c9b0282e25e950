"""Timeline of one bitplane_gemv_kernel launch (dpq_gemv) from per-CTA
%globaltimer stamps (diagnostics hook dpq_debug_gemv_stamps).

    python tools/gv_stamps.py [--shape 4096x4096] [--bits 3]

Needs a -DDPQ_GV_STAMPS build (DPQ_BUILD_DEFINES). Columns (us from the earliest CTA entry; max / median over CTAs): entry,
init done, producer base issued, x staged, LUTs built, first task done,
last task done, last tile epilogue.
"""

from __future__ import annotations

import argparse
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2508_06041_b200 import _lib  # noqa: E402
from paper_2508_06041_b200 import quant as Q  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="4096x4096")
    ap.add_argument("--bits", type=int, default=3)
    ap.add_argument("--dynamic", action="store_true", help="dpq_select_gemv, pair (bits, bits + 1), k=64 f16 G")
    args = ap.parse_args()
    rows, cols = (int(v) for v in args.shape.split("x"))
    dev = torch.device("cuda:0")
    n_copy = max(4, int(np.ceil(300e6 / (rows * cols * args.bits / 8))))
    gen = torch.Generator(device=dev).manual_seed(1)
    rng = np.random.default_rng(0)
    specs = []
    for _ in range(n_copy):
        codes = torch.randint(0, 256, (rows, cols), dtype=torch.uint8, device=dev, generator=gen)
        specs.append((codes, (-rng.random(rows) - 0.5).astype(np.float32),
                      (rng.random(rows) + 0.5).astype(np.float32), 8, 3))
    ds = Q.DeviceStore.from_device_codes(specs, dev)
    x = torch.randn(cols, device=dev)
    y = torch.empty(rows, device=dev)
    lib = _lib.load()
    G = torch.cuda.get_device_properties(0).multi_processor_count
    buf = torch.zeros(G * 8 + G * 64 * 4, dtype=torch.int64, device=dev)
    if args.dynamic:
        from paper_2508_06041_b200 import estimator as E
        from paper_2508_06041_b200 import model as M
        from paper_2508_06041_b200 import runtime as R
        b = args.bits
        pls = []
        for i in range(n_copy):
            Gm = np.random.default_rng(100 + i).standard_normal((64, cols)) / np.sqrt(cols)
            est = float(np.linalg.norm(Gm @ x.cpu().numpy().astype(np.float64)))
            eo = E.ErrorEstimator(E.ProjectionEstimator(Gm, 64, 0), E.IMMEDIATE, (b, b + 1))
            pls.append(R.PlanLayer(M.LayerId(i, "q"), b + 1, b + 0.5, (b, b + 1), est * 0.9, 0.5, eo))
        dp = R.DevicePlan(ds, pls, "f16")

    def call(i):
        if args.dynamic:
            _lib.call("dpq_select_gemv", dp.handle, i, C.c_void_p(x.data_ptr()), None, C.c_void_p(y.data_ptr()),
                      None, None, None, None)
        else:
            _lib.call("dpq_gemv", ds.handle, i, args.bits, C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()), None)
    for i in range(n_copy):                                   # warm (scratch, attributes)
        call(i)
    torch.cuda.synchronize()
    res = []
    for i in range(n_copy):
        buf.zero_()
        _lib.call("dpq_debug_gemv_stamps", C.c_void_p(buf.data_ptr()))
        call(i)
        torch.cuda.synchronize()
        _lib.call("dpq_debug_gemv_stamps", None)
        allb = buf.cpu().numpy().astype(np.float64)
        st = allb[:G * 8].reshape(G, 8)
        ch = allb[G * 8:].reshape(G, 64, 4)
        used = st[:, 0] > 0
        st = st[used]
        t0 = st[:, 0].min()
        rel = np.where(st > 0, (st - t0) / 1e3, np.nan)
        res.append((np.nanmax(rel, axis=0), np.nanmedian(rel, axis=0)))
        if i == n_copy // 2:
            c0 = ch[0]
            ok = c0[:, 0] > 0
            print("CTA 0 chunks (us from first entry): issued landed-read released(last warp)")
            for j in np.nonzero(ok)[0][:48]:
                print(f"  {j:3d} " + " ".join(f"{(v - t0) / 1e3:7.2f}" if v > 0 else "    nan" for v in c0[j, :3]))
    mx = np.median([r[0] for r in res], axis=0)
    md = np.median([r[1] for r in res], axis=0)
    names = ["entry", "init", "base-issued", "x-staged", "lut", "decision", "last-task", "epilogue"]
    print(f"{args.shape} b={args.bits}: us from first entry (median over {n_copy} launches)")
    print("       " + " ".join(f"{n:>11}" for n in names))
    print("max    " + " ".join(f"{v:11.2f}" for v in mx))
    print("median " + " ".join(f"{v:11.2f}" for v in md))
    del lib
    ds.close()


if __name__ == "__main__":
    main()
