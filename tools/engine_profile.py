"""Per-stage timing of the persistent decode engine from %globaltimer stamps.

    python tools/engine_profile.py [--config llama3_8b] [--steps 32] [--static BIT]

Each CTA stamps every stage when it leaves the grid barrier and before it
arrives at the next one; the critical-path time of stage k is
max_c end[k] - max_c end[k-1] (last arrival to last arrival). Op stages are
reported with their algorithmic bytes (planes at the selected bits + lo/span
+ x + y + fp16 G of the estimators fed... counted per consumer)
and achieved GB/s.
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import sys
import time

os.environ.setdefault("DPQ_DEBUG_TIMES", "1")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402


def main():
    import torch
    from paper_2508_06041_b200 import _lib, synth  # noqa: F401
    from paper_2508_06041_b200 import runtime as R
    import bench as B

    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="llama3_8b")
    ap.add_argument("--steps", type=int, default=32)
    ap.add_argument("--target", type=float, default=3.5)
    ap.add_argument("--static", type=int, default=0, help="sentinel-static plan at this bit")
    ap.add_argument("--json", default="")
    ap.add_argument("--dump", default="", help="save raw stamps (npz) for offline analysis")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    cfg, n_bits, b_min = B.model_config(args.config)
    weights, store, _ = synth.random_device_model(cfg, n_bits, b_min, seed=1234)
    ids = store.ordered_ids()
    pairs, prefill, high = B.pairs_for_target(store, args.target)
    if args.static:
        plan = R.sentinel_static_plan({l: args.static for l in ids}, store.param_counts(), float(args.static))
    else:
        plan = synth.projection_plan(store, pairs, prefill, k=64, seed=0, target=args.target)
        calib = np.random.default_rng(7).integers(0, cfg.vocab, 24)
        synth.calibrate_thresholds(weights, store, plan, calib, high_rate=high)
    eng = R.DecodeEngine(weights, store, plan, g_dtype="f16")
    assert eng.persistent, "engine not selected"
    eng.prefill(np.random.default_rng(11).integers(0, cfg.vocab, 16))
    eng.decode_greedy(4)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    eng.decode_greedy(args.steps)
    dt = (time.perf_counter() - t0) / args.steps
    n = C.c_int()
    _lib.call("dpq_session_engine_stages", eng._h, C.byref(n), None, None)
    kinds = np.zeros(n.value, dtype=np.int32)
    idx = np.zeros(n.value, dtype=np.int32)
    _lib.call("dpq_session_engine_stages", eng._h, C.byref(n), C.c_void_p(kinds.ctypes.data),
              C.c_void_p(idx.ctypes.data))
    per = C.c_int()
    _lib.call("dpq_session_debug_times", eng._h, None, 0, C.byref(per))
    G = torch.cuda.get_device_properties(0).multi_processor_count
    rec = per.value // G
    buf = np.zeros(n.value * G * rec, dtype=np.uint64)
    _lib.call("dpq_session_debug_times", eng._h, C.c_void_p(buf.ctypes.data), buf.size, C.byref(per))
    full = buf.reshape(n.value, G, rec)
    st = full[..., :8].astype(np.float64)
    wst = full[..., 8:88].reshape(n.value, G, 16, 5)
    pst = full[..., 88:96]
    cst = full[..., 96:128]
    if args.dump:
        np.savez(args.dump, st=st, wst=wst, pst=pst, cst=cst, kinds=kinds, idx=idx)
    start, end = st[..., 0], st[..., 7]
    pro, loop = st[..., 4], st[..., 5]
    last_end = end.max(axis=1)
    crit = np.diff(np.concatenate([[start[0].min()], last_end])) / 1e3   # us
    # selected bits of the last step
    last = eng.trace.steps[-1]
    bits = [last.bits[l] for l in ids]
    by = B.op_bytes(store, plan, bits, ids, 2)
    names = {0: "begin", 1: "op", 2: "attn", 3: "head", 4: "emit"}
    opn = ["qkv", "o", "upgate", "down"]
    rows = []
    oi = 0
    for k in range(n.value):
        nm = names[int(kinds[k])]
        b = None
        if kinds[k] == 1:
            nm = opn[oi % 4]
            b = float(by[oi])
            oi += 1
        if kinds[k] == 1:
            ph = ((pro[k] - start[k]).mean() / 1e3, (loop[k] - pro[k]).mean() / 1e3, (end[k] - loop[k]).mean() / 1e3,
                  (end[k] - start[k]).max() / 1e3, (start[k].max() - start[k].min()) / 1e3)
        else:
            ph = (0, 0, 0, (end[k] - start[k]).max() / 1e3, (start[k].max() - start[k].min()) / 1e3)
        rows.append((nm, crit[k], b, (end[k] - start[k]).mean() / 1e3, ph))
    tot = crit.sum()
    agg = {}
    for nm, t, b, busy, ph in rows:
        a = agg.setdefault(nm, [0.0, 0.0, 0, 0.0, np.zeros(5)])
        a[0] += t
        a[1] += b or 0.0
        a[2] += 1
        a[3] += busy
        a[4] += np.array(ph)
    print(f"step (host timed, decode_greedy): {dt * 1e3:.3f} ms -> {1 / dt:.1f} tok/s; "
          f"stage critical path sum {tot:.1f} us; G={G}")
    print(f"{'stage':>8} {'n':>4} {'us/stage':>9} {'share':>6} {'GB/s':>8} {'busy':>6} "
          f"{'prolog':>6} {'items':>6} {'combine':>7} {'maxbusy':>7} {'spread':>6}")
    for nm, (t, b, c, busy, ph) in agg.items():
        gbs = b / (t * 1e-6) / 1e9 if b else float("nan")
        ph = ph / c
        print(f"{nm:>8} {c:>4} {t / c:9.2f} {t / tot:6.1%} {gbs:8.1f} {busy / c:6.2f} "
              f"{ph[0]:6.2f} {ph[1]:6.2f} {ph[2]:7.2f} {ph[3]:7.2f} {ph[4]:6.2f}")
    # op phase breakdown (stamps 0..7), mean over CTAs that had work, per op kind
    print("op phases (mean us from barrier release): decide build tabs lut items combine end")
    oi = 0
    ph_acc = {}
    for k in range(n.value):
        if kinds[k] != 1:
            continue
        nm = opn[oi % 4]
        oi += 1
        s_ = st[k]
        ok = s_[:, 5] > 0
        rel = (s_[ok] - s_[ok][:, :1]) / 1e3
        ph_acc.setdefault(nm, []).append(rel.mean(axis=0))
    for nm, v in ph_acc.items():
        v = np.mean(v, axis=0)
        print(f"{nm:>8} " + " ".join(f"{x:6.2f}" for x in v[1:]))
    opb = sum(r[2] for r in rows if r[2])
    rows = [r[:4] for r in rows]
    opt = sum(r[1] for r in rows if r[2])
    print(f"ops: {opb / 1e9:.3f} GB in {opt:.1f} us -> {opb / (opt * 1e-6) / 1e9:.1f} GB/s")
    if args.json:
        json.dump({"step_ms": dt * 1e3, "stages": rows, "op_bytes": opb, "op_us": opt}, open(args.json, "w"))


if __name__ == "__main__":
    main()
