"""Per-stage timeline of the barrier-free engine from its %globaltimer stamps
(DPQ_DEBUG_TIMES=1; the last step of a decode_greedy run).

    python tools/stage_stamps.py [--config llama3_8b] [--static BIT]

Stamps per (stage, CTA): [0] stage entered, [1] input window ready,
[2] LUT + feeds done, [3] plane stream done, [4] reduce duty done, [7] end.
Printed per op kind: mean phase durations over CTAs and the critical path
(last CTA's end of stage k minus last CTA's end of stage k - 1).
"""

from __future__ import annotations

import argparse
import ctypes as C
import os
import sys
import time

os.environ.setdefault("DPQ_DEBUG_TIMES", "1")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402


def main():
    import torch
    from paper_2508_06041_b200 import _lib, synth
    from paper_2508_06041_b200 import runtime as R
    import bench as B

    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="llama3_8b")
    ap.add_argument("--steps", type=int, default=16)
    ap.add_argument("--target", type=float, default=3.5)
    ap.add_argument("--static", type=int, default=0)
    ap.add_argument("--dump", default="")
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
    st = buf.reshape(n.value, G, rec).astype(np.float64)
    if args.dump:
        np.savez(args.dump, st=st, kinds=kinds, idx=idx)
    t_origin = st[0, :, 0].min()
    # end of a stage: op stages -> reducer done [7]; begin / head -> consumers done [4]
    is_op = kinds == 1
    end = np.where(is_op[:, None], st[..., 7], st[..., 4])
    last_end = end.max(axis=1)
    crit = np.diff(np.concatenate([[t_origin], last_end])) / 1e3
    print(f"step {dt * 1e3:.3f} ms -> {1 / dt:.1f} tok/s; stage critical path sum {crit.sum():.1f} us")
    opn = ["qkv", "o", "upgate", "down"]
    agg = {}
    oi = 0
    cols = (0, 1, 2, 3, 4, 7, 5, 6)
    for k in range(n.value):
        if kinds[k] == 1:
            nm = opn[oi % 4]
            oi += 1
            s = st[k]
            ref = last_end[k - 1]
            absx = np.array([(s[:, j].max() - ref) / 1e3 for j in cols])
            mean = np.array([(s[:, j].mean() - ref) / 1e3 for j in cols])
        else:
            nm = {0: "begin", 3: "head"}.get(int(kinds[k]), str(kinds[k]))
            absx = mean = np.zeros(len(cols))
        a = agg.setdefault(nm, [0, 0.0, np.zeros(len(cols)), np.zeros(len(cols))])
        a[0] += 1
        a[1] += crit[k]
        a[2] += absx
        a[3] += mean
    print("stamps rel. to the previous stage's end (us): cons-start input lut base cons-done reducer-done"
          " | producer: base-issued decided")
    for nm, (c, t, ab, mn) in agg.items():
        print(f"{nm:>7} {c:3d} crit {t / c:7.2f} | max " + " ".join(f"{v:6.2f}" for v in ab / c)
              + " | mean " + " ".join(f"{v:6.2f}" for v in mn / c))
    if rec >= 20:
        # reducer warp phases: [16] decide start, [17] decided, [18] statistics, [19] first unit out, [7] done
        print("reducer (max | mean over CTAs, us rel. prev stage end): decide-start first-poll feeds-done(CTA) decided stats first-unit done"
              + (" G.x-words-complete sumsq-words-complete poll-exit decide-return" if rec >= 28 else ""))
        oi = 0
        ragg = {}
        for k in range(n.value):
            if kinds[k] != 1:
                continue
            nm = opn[oi % 4]
            oi += 1
            s = st[k]
            ref = last_end[k - 1]
            cols_r = (16, 22, 20, 17, 18, 19, 7) + ((24, 25, 26, 27) if rec >= 28 else ())
            mx = np.array([(s[:, j][s[:, j] > 0].max() - ref) / 1e3 if np.any(s[:, j] > 0) else 0 for j in cols_r])
            mn = np.array([(s[:, j][s[:, j] > 0].mean() - ref) / 1e3 if np.any(s[:, j] > 0) else 0 for j in cols_r])
            a_ = ragg.setdefault(nm, [0, np.zeros(len(cols_r)), np.zeros(len(cols_r)), 0.0])
            a_[3] += float(np.mean(buf.reshape(n.value, G, rec)[k][:, 23].astype(np.float64)))
            a_[0] += 1
            a_[1] += mx
            a_[2] += mn
        for nm, (c, mx, mn, npoll) in ragg.items():
            print(f"{nm:>7} max " + " ".join(f"{v:6.2f}" for v in mx / c) + " | mean " + " ".join(f"{v:6.2f}" for v in mn / c)
                  + f" | polls {npoll / c:.1f}")
    if rec >= 12:
        # attention units (qkv stages): stamps [8] enter, [9] q ready, [10] rows ready, [11] published
        oi, acc, nq = 0, np.zeros(6), 0
        for k in range(n.value):
            if kinds[k] != 1:
                continue
            if oi % 4 == 1:
                s = st[k]
                ok = s[:, 8] > s[:, 0]
                ref = last_end[k - 1]
                acc += np.array([(s[ok, 0].max() - ref), (s[ok, 1].max() - ref), (s[ok, 8].max() - ref),
                                 (s[ok, 9].max() - ref), (s[ok, 10].max() - ref), (s[ok, 11].max() - ref)]) / 1e3
                nq += 1
            oi += 1
        print("attention CTAs (o stage), max stamps rel. prev end: cons-start input-ready enter q-ready rows-ready published")
        print("        " + " ".join(f"{v:6.2f}" for v in acc / max(nq, 1)))
        # clock64 deltas (cycles) inside the unit, last qkv stage
        k = [i for i in range(n.value) if kinds[i] == 1][-3]
        s = buf.reshape(n.value, G, rec)[k]
        ok = s[:, 8] > s[:, 0]
        print("attention unit cycles (median over units): tma-issued q-ready rows-ready scores-done published")
        print("        " + " ".join(f"{int(np.median(s[ok, j].astype(np.int64)))}" for j in (12, 13, 14, 15, 6)))


if __name__ == "__main__":
    main()
