"""Per-phase timing of the fused op kernel from %globaltimer stamps.

    DPQ_DEBUG_TIMES=1 python tools/profile_op.py [--blocks 4] [--static] [--graph]

Stamps (per CTA): 0 start, 1 after griddepcontrol.wait, 2 LUT built,
3 estimator partials + barrier arrive, 4 decider done (last CTA) / passed,
5 before decision wait, 6 after decision wait, 7 end.
"""

from __future__ import annotations

import argparse
import ctypes as C
import os
import sys

os.environ.setdefault("DPQ_DEBUG_TIMES", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2508_06041_b200 import _lib, synth  # noqa: E402
from paper_2508_06041_b200 import model as M  # noqa: E402
from paper_2508_06041_b200 import runtime as R  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--blocks", type=int, default=4)
    ap.add_argument("--static", action="store_true")
    ap.add_argument("--graph", action="store_true", help="time a graph step instead of an eager one")
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--eager", action="store_true", help="no CUDA graph (for ncu)")
    args = ap.parse_args()
    cfg = M.ModelConfig(args.blocks, 4096, 32, 14336, vocab=256, seq_cap=256, n_kv_heads=8)
    w, store, _ = synth.random_device_model(cfg, 4, 3, seed=1)
    ids = store.ordered_ids()
    if args.static:
        plan = R.sentinel_static_plan({l: 4 for l in ids}, store.param_counts(), 4.0)
    else:
        plan = synth.projection_plan(store, {l: (3, 4) for l in ids}, {l: 4 for l in ids}, k=64)
        synth.calibrate_thresholds(w, store, plan, np.arange(24) % 256, high_rate=0.5)
    eng = R.DecodeEngine(w, store, plan, use_graph=not args.eager)
    eng.prefill(np.arange(8))
    for t in range(args.steps):
        eng.step(t + 10, dynamic=True, want_logits=False)
    n_ops = 4 * cfg.n_blocks
    op_ms = np.zeros(n_ops, dtype=np.float32)
    nout = C.c_int()
    per0 = C.c_int()
    _lib.call("dpq_session_debug_times", eng._h, None, -1, C.byref(per0))
    if args.graph:
        eng.step(99, dynamic=True)
    else:
        _lib.call("dpq_session_profile_ops", eng._h, 99, 1, C.c_void_p(op_ms.ctypes.data), n_ops,
                  C.byref(nout))
    per = C.c_int()
    _lib.call("dpq_session_debug_times", eng._h, None, 0, C.byref(per))
    buf = np.zeros(n_ops * 2 * per.value, dtype=np.uint64)
    _lib.call("dpq_session_debug_times", eng._h, C.c_void_p(buf.ctypes.data), buf.size, C.byref(per))
    buf = buf.reshape(-1, per.value // 8, 8).astype(np.int64)
    names = ["qkv", "o", "upgate", "down"]
    os.makedirs("gpurun_out", exist_ok=True)
    np.save(f"gpurun_out/stamps_{'static' if args.static else 'dyn'}_{'graph' if args.graph else 'eager'}.npy", buf)
    valid_all = buf[buf[:, :, 0] > 0]
    T0 = valid_all[:, 0].min() if len(valid_all) else 0
    print("timeline (us from first stamp): op first_start last_start median_dep_ready last_end")
    for i in range(n_ops):
        t = buf[i][buf[i][:, 0] > 0]
        if len(t) == 0:
            continue
        print(f"  {names[i % 4] + str(i // 4):>10} {(t[:, 0].min() - T0) / 1e3:8.1f} {(t[:, 0].max() - T0) / 1e3:8.1f} "
              f"{(np.median(t[:, 1]) - T0) / 1e3:8.1f} {(t[:, 7].max() - T0) / 1e3:8.1f}")
    print(f"{'op':>10} {'ev_us':>7} {'grid':>4} {'start_spread':>12} {'wait':>6} {'lut':>6} {'G+arr':>6} "
          f"{'->dec':>6} {'phA':>6} {'dwait':>6} {'rest':>6} {'total':>7}")
    for i in range(n_ops):
        t = buf[i]
        valid = t[:, 0] > 0
        t = t[valid]
        if len(t) == 0:
            continue
        t0 = t[:, 0].min()
        d = lambda a, b: np.median(np.where((t[:, a] > 0) & (t[:, b] > 0), t[:, b] - t[:, a], 0)) / 1e3
        total = (t[:, 7].max() - t0) / 1e3
        spread = (t[:, 0].max() - t0) / 1e3
        has5 = (t[:, 5] > 0).any()
        phA = d(4, 5) if has5 else d(4, 7)
        dw = d(5, 6) if has5 else 0.0
        rest = d(6, 7) if has5 else 0.0
        print(f"{names[i % 4] + str(i // 4):>10} {op_ms[i] * 1e3 if nout.value else 0:7.1f} {len(t):4d} "
              f"{spread:12.1f} {d(0, 1):6.1f} {d(1, 2):6.1f} {d(2, 3):6.1f} {d(3, 4):6.1f} {phA:6.1f} "
              f"{dw:6.1f} {rest:6.1f} {total:7.1f}")
        last = t[:, 4].argmax()
        print(f"{'':>10} last CTA decider: {(t[last, 4] - t[last, 3]) / 1e3:.1f} us; "
              f"max end-start per CTA: {((t[:, 7] - t[:, 0]).max()) / 1e3:.1f} us; "
              f"min: {((t[:, 7] - t[:, 0]).min()) / 1e3:.1f} us")


if __name__ == "__main__":
    main()
