"""Where does the selector overhead go? Times single-step launches of the
persistent engine (8B-shaped, DP 3.5-bit) three ways on the same tokens:

  dynamic  - estimator feeds + decisions + base pass / extra pass split;
  forced   - the same per-layer bits replayed (C.force): feeds still run, but
             every plane of a layer is a base plane (one pass, no decision wait);
  static   - sentinel plans at 3 and 4 bits (no feeds, one pass), interpolated
             at the realized bits.

    python tools/selector_split.py [--steps 48]
"""

from __future__ import annotations

import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench as B  # noqa: E402
from paper_2508_06041_b200 import runtime as R, synth  # noqa: E402


def timed_steps(eng, toks, forced=None):
    ts = []
    for i, t in enumerate(toks):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        eng.step(int(t), dynamic=True, want_logits=False,
                 forced_bits=None if forced is None else forced[i])
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return np.array(ts) * 1e3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=48)
    args = ap.parse_args()
    torch.cuda.set_device(0)
    cfg, n_bits, b_min = B.model_config("llama3_8b")
    w, store, _ = synth.random_device_model(cfg, n_bits, b_min, seed=1234)
    pairs, prefill, high = B.pairs_for_target(store, 3.5)
    plan = synth.projection_plan(store, pairs, prefill, k=64, seed=0, target=3.5)
    synth.calibrate_thresholds(w, store, plan, np.random.default_rng(7).integers(0, cfg.vocab, 48),
                               high_rate=high)
    ids = store.ordered_ids()
    prompt = np.random.default_rng(11).integers(0, cfg.vocab, 16)
    toks = np.random.default_rng(12).integers(0, cfg.vocab, args.steps)
    eng = R.DecodeEngine(w, store, plan, g_dtype="f16")
    eng.prefill(prompt)
    t_dyn = timed_steps(eng, toks)
    recs = eng.trace.steps[-args.steps:]
    bits = [np.array([r.bits[l] for l in ids], dtype=np.int8) for r in recs]
    eff = float(np.mean([r.effective_bits for r in recs]))
    eng.reset()
    eng.prefill(prompt)
    t_forced = timed_steps(eng, toks, bits)
    eng.close()
    st = {}
    for b in (3, 4):
        sp = R.sentinel_static_plan({l: b for l in ids}, store.param_counts(), float(b))
        e2 = R.DecodeEngine(w, store, sp)
        e2.prefill(prompt)
        st[b] = timed_steps(e2, toks)
        e2.close()
    # heterogeneous bits without any estimator: a (3, 4) plan with T = +inf on
    # every layer (no feeds, no decisions), the recorded bits replayed
    nofeed = R.PrecisionPlan("nofeed", 3.5, float("nan"),
                             {l: R.PlanLayer(l, 4, 3.5, (3, 4), np.inf, 1.0, None) for l in ids},
                             store.param_counts())
    e3 = R.DecodeEngine(w, store, nofeed)
    e3.prefill(prompt)
    t_nofeed = timed_steps(e3, toks, bits)
    e3.close()
    s3, s4 = np.median(st[3][8:]), np.median(st[4][8:])
    nf = np.median(t_nofeed[8:])
    print(f"forced replay without estimators (no feeds): {nf:.3f} ms "
          f"({100 * (nf / (s3 + (s4 - s3) * (eff - 3)) - 1):.1f}% over static)")
    s_interp = s3 + (s4 - s3) * (eff - 3)
    d, f = np.median(t_dyn[8:]), np.median(t_forced[8:])
    print(f"single-step launches, median of {args.steps - 8} (ms): dynamic {d:.3f}  forced-replay {f:.3f}  "
          f"static3 {s3:.3f} static4 {s4:.3f} -> static at {eff:.3f} bits {s_interp:.3f}")
    print(f"overhead vs static: dynamic {100 * (d / s_interp - 1):.1f}%  forced {100 * (f / s_interp - 1):.1f}%  "
          f"(forced isolates the feeds; dynamic - forced = decision wait + two-pass split)")


if __name__ == "__main__":
    main()
