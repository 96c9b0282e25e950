"""Generate tests/golden/ fixtures by running the UNMODIFIED reference.

Run in the build container (where /root/reference exists):

    python tools/make_golden.py

The reference is imported read-only from /root/reference/pkg/src. Outputs are
small .npz/.json fixtures that travel to the GPU box (the reference does not).
Shipped reference plans are copied verbatim as data fixtures (they carry the
calibrated G matrices the report numbers depend on).
"""

from __future__ import annotations

import json
import os
import shutil
import sys

import numpy as np

REF = "/root/reference/pkg"
sys.path.insert(0, os.path.join(REF, "src"))

from dpq import estimator as E  # noqa: E402
from dpq import model as M  # noqa: E402
from dpq import planner as P  # noqa: E402
from dpq import quant as Q  # noqa: E402
from dpq import runtime as R  # noqa: E402
from dpq import sensitivity as S  # noqa: E402
from dpq.corpus import contiguous_chunks, generate_text, sample_chunks  # noqa: E402
from dpq.fitter import FitConfig  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                   "tests", "golden")


def lname(lid):
    return lid.name


def quant_vectors():
    """Known-answer vectors for the nested store (quant.py)."""
    out = {}
    W = np.array([[0.0, 0.3, 0.6, 1.0]])
    q = Q.quantize_layer(W, 2, 2)
    out["kat2_codes"] = q.codes
    out["kat2_deq"] = Q.dequantize(q, 2)
    rng = np.random.default_rng(1234)
    cases = [(37, 53, 6, 3), (64, 96, 8, 3), (32, 512, 4, 3), (8, 16, 6, 3),
             (1, 4, 6, 3), (48, 512, 6, 2)]
    for i, (r, c, n, bmin) in enumerate(cases):
        W = rng.normal(0.0, 1.0 / np.sqrt(c), (r, c)).astype(np.float32)
        if i == 0:
            W[3, :] = 0.25          # degenerate row (span 0)
        q = Q.quantize_layer(W, n, bmin)
        x = rng.normal(size=c)
        if r * c <= 8192:
            out[f"c{i}_W"] = W
        out[f"c{i}_meta"] = np.array([r, c, n, bmin])
        out[f"c{i}_codes"] = q.codes
        out[f"c{i}_lo"] = q.lo
        out[f"c{i}_hi"] = q.hi
        out[f"c{i}_x"] = x
        for b in range(bmin, n + 1):
            out[f"c{i}_deq{b}"] = Q.dequantize(q, b) if r * c <= 4096 else np.zeros(0)
            out[f"c{i}_y{b}"] = Q.gemv(q, b, x)
        if n > bmin:
            out[f"c{i}_exact"] = np.array([E.exact_error(q, bmin, bmin + 1, x)])
        out[f"c{i}_packed"] = np.frombuffer(Q.pack_codes(q.codes, n), dtype=np.uint8)
    np.savez_compressed(os.path.join(OUT, "quant_vectors.npz"), **out)


def toy_pipeline():
    """configs/toy.json pipeline: store hash, shipped plans, eval + decode
    traces through the reference DecodeEngine."""
    cfg = json.load(open(os.path.join(REF, "configs", "toy.json")))
    mc = M.ModelConfig.from_dict(cfg["model"])
    weights = M.init_model(cfg["seed"], mc)
    store = Q.quantize_model(weights, cfg["quant"]["n_bits"], cfg["quant"]["b_min"])
    tmp = "/tmp/_golden_store.dpqs"
    Q.save_store(store, tmp)
    store_hash = Q.file_hash(tmp)
    shutil.copyfile(os.path.join(REF, "data", "toy.txt"), os.path.join(OUT, "toy_corpus.txt"))
    tokens = np.frombuffer(open(os.path.join(REF, "data", "toy.txt"), "rb").read(),
                           dtype=np.uint8).astype(np.int64)
    e = cfg["eval"]
    chunks = contiguous_chunks(tokens, e["seq_len"], e["n_samples"], e["offset"])
    os.makedirs(os.path.join(OUT, "plans"), exist_ok=True)
    summary = {"config": cfg["model"], "n_bits": cfg["quant"]["n_bits"],
               "b_min": cfg["quant"]["b_min"], "seed": cfg["seed"],
               "store_hash": store_hash, "weights_checksum": weights.checksum(),
               "eval": e, "plans": {}}
    # fp row (report.csv:2)
    losses = []
    for toks in chunks:
        _, tr = R.eval_perplexity(weights, store, toks, "fp")
        losses.extend(tr.token_losses)
    summary["fp_perplexity"] = float(np.exp(np.mean(losses)))

    traces = {}
    for name in ("dp_t3.5", "dp_t4", "llm_mq_t3.5", "hawq_v2_t4"):
        src = os.path.join(REF, "artifacts", "plans", name + ".json")
        shutil.copyfile(src, os.path.join(OUT, "plans", name + ".json"))
        plan = R.load_plan(src, store)
        ls, effs, ops = [], [], 0
        for ci, toks in enumerate(chunks):
            ppl, tr = R.eval_perplexity(weights, store, toks, "dynamic", plan=plan,
                                        store_hash=store_hash)
            ls.extend(tr.token_losses)
            effs.append(tr.mean_effective_bits())
            ops += tr.estimator_ops
            if ci == 0:
                traces[name] = tr
        summary["plans"][name] = {
            "perplexity": float(np.exp(np.mean(ls))),
            "effective_bits": float(np.mean(effs)),
            "estimator_ops": int(ops)}

    # per-step trace of chunk 0 for each plan: bits / estimates / losses
    tv = {}
    for name, tr in traces.items():
        lids = list(tr.steps[0].bits)
        tv[f"{name}_layers"] = np.array([lname(l) for l in lids])
        tv[f"{name}_bits"] = np.array([[s.bits[l] for l in lids] for s in tr.steps])
        tv[f"{name}_est"] = np.array([[np.nan if s.estimates[l] is None else s.estimates[l]
                                       for l in lids] for s in tr.steps])
        tv[f"{name}_losses"] = np.array(tr.token_losses)
        tv[f"{name}_eff"] = np.array([s.effective_bits for s in tr.steps])

    # greedy decode with logits per step (dp_t3.5)
    plan = R.load_plan(os.path.join(OUT, "plans", "dp_t3.5.json"), store)
    prompt = tokens[:16]
    eng = R.DecodeEngine(weights, store, plan, store_hash)
    logits = eng.prefill(prompt)
    lg, toks_out = [logits], []
    for _ in range(24):
        nxt = int(np.argmax(logits))
        toks_out.append(nxt)
        logits = eng.step(nxt, dynamic=True)
        lg.append(logits)
    tv["decode_prompt"] = prompt
    tv["decode_tokens"] = np.array(toks_out)
    tv["decode_logits"] = np.array(lg)
    lids = list(eng.trace.steps[0].bits)
    tv["decode_layers"] = np.array([lname(l) for l in lids])
    tv["decode_bits"] = np.array([[s.bits[l] for l in lids] for s in eng.trace.steps])
    tv["decode_est"] = np.array([[np.nan if s.estimates[l] is None else s.estimates[l]
                                  for l in lids] for s in eng.trace.steps])
    summary["decode_estimator_ops"] = int(eng.trace.estimator_ops)

    # exact-mode + async plan built by the reference planner (as in
    # tests/test_runtime.py:323-341), evaluated with both async rules and
    # track_exact.
    calib = sample_chunks(tokens, cfg["calib"]["seq_len"], cfg["calib"]["n_samples"],
                          seed=cfg["calib"]["seed"])
    prof = S.profile(weights, store, calib)
    planx, _, _ = P.build_dp_plan(weights, store, prof, calib, 5.0, 4.0,
                                  estimator_mode="exact", use_async=True,
                                  hyper=FitConfig(epochs=1), store_hash=store_hash)
    R.save_plan(planx, os.path.join(OUT, "plans", "exact_async_t4.json"))
    planx = R.load_plan(os.path.join(OUT, "plans", "exact_async_t4.json"), store)
    for rule in ("prev_step", "prev_block"):
        ppl, tr = R.eval_perplexity(weights, store, chunks[0], "dynamic", plan=planx,
                                    store_hash=store_hash, track_exact=True,
                                    async_rule=rule)
        lids = list(tr.steps[0].bits)
        tv[f"exact_{rule}_layers"] = np.array([lname(l) for l in lids])
        tv[f"exact_{rule}_bits"] = np.array([[s.bits[l] for l in lids] for s in tr.steps])
        tv[f"exact_{rule}_est"] = np.array(
            [[np.nan if s.estimates[l] is None else s.estimates[l] for l in lids]
             for s in tr.steps])
        xl = list(tr.steps[0].exact_errors)
        tv[f"exact_{rule}_xlayers"] = np.array([lname(l) for l in xl])
        tv[f"exact_{rule}_xerr"] = np.array([[s.exact_errors[l] for l in xl]
                                             for s in tr.steps])
        tv[f"exact_{rule}_losses"] = np.array(tr.token_losses)
        summary[f"exact_{rule}_perplexity"] = ppl
        summary[f"exact_{rule}_estimator_ops"] = int(tr.estimator_ops)
        cmp = R.incurred_error_comparison(tr, planx)
        summary[f"exact_{rule}_incurred"] = {l.name: list(v) for l, v in cmp.items()}

    # linear-estimator plan: dp_t3.5 with every projection swapped for a
    # LinearEstimator (slope from the layer's first step estimate).
    planl = R.load_plan(os.path.join(OUT, "plans", "dp_t3.5.json"), store)
    for i, (lid, pl) in enumerate(sorted(planl.layers.items(),
                                         key=lambda kv: (kv[0].block, M.KINDS.index(kv[0].kind)))):
        if pl.estimator is not None:
            cols = store.layers[lid].shape[1]
            slope = pl.T / np.sqrt(cols) * (0.9 + 0.1 * (i % 3))
            pl.estimator = E.ErrorEstimator(
                E.LinearEstimator(float(slope), 0.001 * ((i % 5) - 2), 0.95),
                pl.estimator.input_source, pl.estimator.pair)
    R.save_plan(planl, os.path.join(OUT, "plans", "linear_t3.5.json"))
    ppl, tr = R.eval_perplexity(weights, store, chunks[1], "dynamic", plan=planl,
                                store_hash=store_hash)
    lids = list(tr.steps[0].bits)
    tv["linear_layers"] = np.array([lname(l) for l in lids])
    tv["linear_bits"] = np.array([[s.bits[l] for l in lids] for s in tr.steps])
    tv["linear_est"] = np.array([[np.nan if s.estimates[l] is None else s.estimates[l]
                                  for l in lids] for s in tr.steps])
    tv["linear_losses"] = np.array(tr.token_losses)
    summary["linear_perplexity"] = ppl
    summary["linear_estimator_ops"] = int(tr.estimator_ops)
    summary["linear_chunk"] = 1

    np.savez_compressed(os.path.join(OUT, "toy_traces.npz"), **tv)
    with open(os.path.join(OUT, "toy_summary.json"), "w") as f:
        json.dump(summary, f, indent=1)
    print("store hash", store_hash)
    print(json.dumps(summary["plans"], indent=1))


def cfg1_vectors():
    """cfg1 shapes (d=512, d_ff=1792, n=4, b_min=3): weights checksum and
    one layer of each shape's gemv at b=3,4."""
    mc = M.ModelConfig(n_blocks=2, d_model=512, n_heads=8, d_ff=1792, vocab=256,
                       seq_cap=512)
    w = M.init_model(0, mc)
    out = {"weights_checksum": np.array([w.checksum()]),
           "config_hash": np.array([mc.hash()])}
    rng = np.random.default_rng(7)
    for kind in ("q", "up", "down"):
        q = Q.quantize_layer(w.linears[M.LayerId(0, kind)], 4, 3)
        x = rng.normal(size=q.shape[1])
        out[f"{kind}_x"] = x
        out[f"{kind}_lo"] = q.lo
        out[f"{kind}_hi"] = q.hi
        out[f"{kind}_codes_sum"] = np.array([int(q.codes.astype(np.int64).sum())])
        for b in (3, 4):
            out[f"{kind}_y{b}"] = Q.gemv(q, b, x)
    np.savez_compressed(os.path.join(OUT, "cfg1_vectors.npz"), **out)


def calib_vectors():
    """Offline calibration on the reference:
    collect_error_samples (estimator.py:132-165) on a small GQA-free model
    at max bits 5 with (3,4) / (4,5) pairs, and calibrate_projection
    (estimator.py:208-264) of two layers' projections on those samples."""
    mc = M.ModelConfig(n_blocks=2, d_model=64, n_heads=4, d_ff=128, vocab=256, seq_cap=64)
    w = M.init_model(3, mc)
    store = Q.quantize_model(w, 6, 3)
    ids = M.layer_ids(mc)
    pairs = {lid: ((3, 4) if i % 2 == 0 else (4, 5)) for i, lid in enumerate(ids)}
    max_bits = {lid: 5 for lid in ids}
    toks = np.frombuffer(generate_text(1, 4096).encode(), dtype=np.uint8).astype(np.int64)
    calib = sample_chunks(toks, 12, 4, seed=2)
    samples = E.collect_error_samples(w, store, pairs, max_bits, calib)
    out = {"calib": np.array(calib)}
    for lid in ids:
        s = samples[lid]
        out[f"{lid.name}/errors"] = s.errors
        out[f"{lid.name}/norms"] = s.norms
        out[f"{lid.name}/inputs"] = s.inputs
    for lid in (ids[0], ids[6]):
        l, h = pairs[lid]
        est = E.build_projection(store.layers[lid], l, h, 8, 5)
        cal, hist, warn = E.calibrate_projection(est, samples[lid].inputs, samples[lid].errors, epochs=40)
        out[f"{lid.name}/G0"] = est.G
        out[f"{lid.name}/G"] = cal.G
        out[f"{lid.name}/history"] = np.array(hist)
        out[f"{lid.name}/warning"] = np.array([int(warn)])
        lin = E.fit_linear(samples[lid].errors, samples[lid].norms)
        out[f"{lid.name}/linear"] = (np.array([lin.slope, lin.intercept, lin.r2]) if lin is not None
                                     else np.array([np.nan, np.nan, np.nan]))
    np.savez_compressed(os.path.join(OUT, "calib_vectors.npz"), **out)


def cfg1_plan():
    """cfg1 with the reference's own planner: init_model(0),
    quantize_model(4, 3), corpus generate_text(0, 16384), calib
    sample_chunks(32, 8, seed 0), sensitivity profile, build_dp_plan(budget
    4.0, target 3.5, hybrid, k=64, seed 0, calibrate=True) with the toy
    config's fit hyper-parameters; the plan JSON plus the reference
    DecodeEngine's greedy decode of 64 tokens from toks[:16]."""
    from dpq.cli import default_alpha
    from dpq import fitter as F
    mc = M.ModelConfig(n_blocks=2, d_model=512, n_heads=8, d_ff=1792, vocab=256, seq_cap=512)
    weights = M.init_model(0, mc)
    store = Q.quantize_model(weights, 4, 3)
    tmp = "/tmp/_golden_cfg1.dpqs"
    Q.save_store(store, tmp)
    store_hash = Q.file_hash(tmp)
    tokens = np.frombuffer(generate_text(0, 16384).encode(), dtype=np.uint8).astype(np.int64)
    calib = sample_chunks(tokens, 32, 8, 0)
    prof = S.profile(weights, store, calib, store_hash=store_hash)
    hyper = F.FitConfig(epochs=5, lr=0.01, alpha=default_alpha(3.5), batch_size=2, seed=0)
    plan, _, _ = P.build_dp_plan(weights, store, prof, calib, 4.0, 3.5, estimator_mode="hybrid",
                                 use_async=False, k=64, seed=0, calibrate=True, hyper=hyper,
                                 store_hash=store_hash)
    os.makedirs(os.path.join(OUT, "plans"), exist_ok=True)
    R.save_plan(plan, os.path.join(OUT, "plans", "cfg1_dp_t3.5.json"))
    out, tr = R.decode(weights, store, plan, tokens[:16], 64, store_hash=store_hash)
    np.savez_compressed(os.path.join(OUT, "cfg1_plan_decode.npz"), tokens=np.array(out),
                        prompt=tokens[:16], eff=np.array([s.effective_bits for s in tr.steps]),
                        store_hash=np.array([store_hash]), avg_p=np.array([P.plan_effective_bits(plan)]))


def model_vectors():
    """model.forward / teacher_forced_loss / backward (model.py:286-460) on a
    toy config, full-precision and 4-bit dequantized providers."""
    mc = M.ModelConfig(n_blocks=2, d_model=32, n_heads=4, d_ff=64, vocab=256, seq_cap=64)
    w = M.init_model(0, mc)
    store = Q.quantize_model(w, 6, 3)
    toks = np.random.default_rng(4).integers(0, 256, 10)
    out = {"tokens": toks}
    for name, prov in (("fp", None), ("q4", lambda lid: Q.dequantize(store.layers[lid], 4))):
        lg, tape = M.forward(w, toks, prov, want_tape=True)
        out[f"{name}/logits"] = lg
        out[f"{name}/x_final"] = tape.x_final
        for b, bt in enumerate(tape.blocks):
            for f in ("n1", "attn_cat", "h", "probs", "x_mid"):
                out[f"{name}/b{b}/{f}"] = getattr(bt, f)
        loss, ppl, per = M.teacher_forced_loss(w, toks, prov)
        out[f"{name}/tfl"] = np.array([loss, ppl])
        out[f"{name}/per_token"] = per
        bl, bundle, _ = M.backward(w, toks, prov)
        out[f"{name}/bwd_loss"] = np.array([bl])
        for lid in M.layer_ids(mc):
            out[f"{name}/wg/{lid.name}"] = bundle.weight_grads[lid]
            out[f"{name}/og/{lid.name}"] = bundle.output_grads[lid]
    np.savez_compressed(os.path.join(OUT, "model_vectors.npz"), **out)


if __name__ == "__main__":
    os.makedirs(OUT, exist_ok=True)
    if len(sys.argv) > 1 and sys.argv[1] == "model":
        model_vectors()
        sys.exit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "calib":
        calib_vectors()
        sys.exit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "cfg1_plan":
        cfg1_plan()
        sys.exit(0)
    quant_vectors()
    cfg1_vectors()
    toy_pipeline()
    calib_vectors()
    cfg1_plan()
    model_vectors()
