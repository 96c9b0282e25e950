"""Decode engine parity on the GPU against the oracle and the reference's
golden traces (mirrors reference tests/test_runtime.py and the hot-path
acceptance criteria C5/C8)."""

import numpy as np
import pytest

from oracle import dpq_oracle as O
from paper_2508_06041_b200 import model as M
from paper_2508_06041_b200 import quant as Q
from paper_2508_06041_b200 import runtime as R

from conftest import plan_path
from helpers import EPS_DECISION, canon, decision_mismatches, oracle_engine, oracle_eval, trace_arrays

pytestmark = pytest.mark.gpu
LOGIT_TOL = 2e-5          # max |dlogit| / max |logit|
LOSS_TOL = 1e-5           # per-token loss, absolute (nats)


def forced_from_oracle(eng_o, ids):
    return [np.array([r.bits[O.key(l)] for l in ids], dtype=np.int8) for r in eng_o.records]


def device_eval_forced(weights, store, plan, tokens, forced, **kw):
    """eval_perplexity with the decisions replayed from `forced` (list per step)."""
    eng = R.DecodeEngine(weights, store, plan, **kw)
    logits = eng.step(int(tokens[0]), dynamic=False)
    losses, all_logits = [], [logits]
    for i in range(1, len(tokens)):
        z = logits - logits.max()
        losses.append(float(np.log(np.exp(z).sum()) - z[tokens[i]]))
        if i < len(tokens) - 1:
            logits = eng.step(int(tokens[i]), dynamic=True, forced_bits=forced[i - 1])
            all_logits.append(logits)
    return losses, eng, np.array(all_logits)


def Ts(plan, ids):
    return np.array([plan.layers[l].T for l in ids], dtype=np.float64)


@pytest.mark.parametrize("name", ["dp_t3.5", "dp_t4", "llm_mq_t3.5", "hawq_v2_t4"])
def test_report_numbers_on_device(report_setup, golden_summary, name):
    """report.csv rows: perplexity / effective bits / estimator ops, with the
    device following the oracle's decisions (forced replay) and the device's
    own decisions checked against the oracle under the eps rule."""
    S = report_setup
    plan = R.load_plan(plan_path(name), S.store)
    ids = canon(S.store.layers)
    T = Ts(plan, ids)
    losses, effs, ops = [], [], 0
    for toks in S.chunks:
        _, ls_o, eng_o = oracle_eval(S.weights, S.store, plan, toks)
        forced = forced_from_oracle(eng_o, ids)
        ls, eng, _ = device_eval_forced(S.weights, S.store, plan, toks, forced, store_hash=S.store_hash,
                                        g_dtype="f32")
        np.testing.assert_allclose(ls, ls_o, atol=LOSS_TOL)
        losses.extend(ls)
        effs.append(eng.trace.mean_effective_bits())
        ops += eng.trace.estimator_ops
        # device estimates vs oracle, and the decisions they imply
        bits_o, est_o = trace_arrays(eng_o.records, ids)
        _, est_d = trace_arrays(eng.trace.steps, ids)
        np.testing.assert_allclose(est_d, est_o, rtol=1e-4, equal_nan=True)
        implied = np.where(np.isnan(est_d), bits_o, np.where(est_d > T, [plan.layers[l].pair[1] for l in ids],
                                                               [plan.layers[l].pair[0] for l in ids]))
        assert not decision_mismatches(implied, bits_o, est_o, T, EPS_DECISION["f32"], until_first=False)
    exp = golden_summary["plans"][name]
    assert float(np.exp(np.mean(losses))) == pytest.approx(exp["perplexity"], rel=1e-6)
    assert float(np.mean(effs)) == pytest.approx(exp["effective_bits"], abs=1e-12)
    assert ops == exp["estimator_ops"]


def test_free_running_dynamic_plan(report_setup, golden_traces):
    """Unforced device run of dp_t3.5: decisions equal the reference's until
    the first tie (|est - T| <= eps |T|), f16 G."""
    S = report_setup
    plan = R.load_plan(plan_path("dp_t3.5"), S.store)
    ppl, tr = R.eval_perplexity(S.weights, S.store, S.chunks[0], "dynamic", plan=plan,
                                store_hash=S.store_hash)
    ids = [M.LayerId.from_name(n) for n in golden_traces["dp_t3.5_layers"]]
    bits_d, _ = trace_arrays(tr.steps, ids)
    bits_r, est_r = golden_traces["dp_t3.5_bits"], golden_traces["dp_t3.5_est"]
    T = Ts(plan, ids)
    for s in range(len(bits_r)):
        bad = decision_mismatches(bits_d[s:s + 1], bits_r[s:s + 1], est_r[s:s + 1], T, EPS_DECISION["f16"])
        assert not bad, bad
        if not np.array_equal(bits_d[s], bits_r[s]):
            break           # a tie: trajectories may diverge from here on
    assert np.isfinite(ppl)


def test_decode_matches_golden(report_setup, golden_traces):
    S = report_setup
    plan = R.load_plan(plan_path("dp_t3.5"), S.store)
    ids = [M.LayerId.from_name(n) for n in golden_traces["decode_layers"]]
    prompt = golden_traces["decode_prompt"]
    gold_toks = golden_traces["decode_tokens"]
    # step API with the reference decisions replayed: logits per step
    eng = R.DecodeEngine(S.weights, S.store, plan, S.store_hash, g_dtype="f32")
    logits = eng.prefill(prompt)
    lg = [logits]
    for s, tok in enumerate(gold_toks):
        logits = eng.step(int(tok), dynamic=True, forced_bits=golden_traces["decode_bits"][s])
        lg.append(logits)
    lg = np.array(lg)
    ref = golden_traces["decode_logits"]
    assert np.max(np.abs(lg - ref)) <= LOGIT_TOL * np.max(np.abs(ref))
    assert [int(np.argmax(v)) for v in lg[:-1]] == gold_toks.tolist()
    # device greedy loop (argmax fed back on the GPU)
    out, tr = R.decode(S.weights, S.store, plan, prompt, len(gold_toks), store_hash=S.store_hash,
                       g_dtype="f32")
    bits_d, _ = trace_arrays(tr.steps, ids)
    if np.array_equal(bits_d, golden_traces["decode_bits"]):
        assert out == gold_toks.tolist()
    assert len(out) == len(gold_toks) == len(tr.steps)


@pytest.mark.parametrize("rule", ["prev_step", "prev_block"])
def test_exact_async_plan_on_device(report_setup, golden_traces, golden_summary, rule):
    S = report_setup
    plan = R.load_plan(plan_path("exact_async_t4"), S.store)
    ids = [M.LayerId.from_name(n) for n in golden_traces[f"exact_{rule}_layers"]]
    forced = list(golden_traces[f"exact_{rule}_bits"].astype(np.int8))
    ls, eng, _ = device_eval_forced(S.weights, S.store, plan, S.chunks[0], forced, track_exact=True,
                                    async_rule=rule, g_dtype="f32")
    np.testing.assert_allclose(ls, golden_traces[f"exact_{rule}_losses"], atol=LOSS_TOL)
    _, est_d = trace_arrays(eng.trace.steps, ids)
    np.testing.assert_allclose(est_d, golden_traces[f"exact_{rule}_est"], rtol=1e-4, atol=1e-9,
                               equal_nan=True)
    xids = [M.LayerId.from_name(n) for n in golden_traces[f"exact_{rule}_xlayers"]]
    xerr = np.array([[r.exact_errors[l] for l in xids] for r in eng.trace.steps])
    np.testing.assert_allclose(xerr, golden_traces[f"exact_{rule}_xerr"], rtol=1e-4, atol=1e-9)
    assert eng.trace.estimator_ops == golden_summary[f"exact_{rule}_estimator_ops"]
    cmp = R.incurred_error_comparison(eng.trace, plan)
    assert cmp
    for dyn, matched, m, n in cmp.values():
        assert 0 <= m <= n


def test_linear_plan_on_device(report_setup, golden_traces, golden_summary):
    S = report_setup
    plan = R.load_plan(plan_path("linear_t3.5"), S.store)
    ids = [M.LayerId.from_name(n) for n in golden_traces["linear_layers"]]
    toks = S.chunks[golden_summary["linear_chunk"]]
    forced = list(golden_traces["linear_bits"].astype(np.int8))
    ls, eng, _ = device_eval_forced(S.weights, S.store, plan, toks, forced, g_dtype="f32")
    np.testing.assert_allclose(ls, golden_traces["linear_losses"], atol=LOSS_TOL)
    _, est_d = trace_arrays(eng.trace.steps, ids)
    np.testing.assert_allclose(est_d, golden_traces["linear_est"], rtol=1e-5, equal_nan=True)
    # unforced: decisions identical outside eps
    _, tr = R.eval_perplexity(S.weights, S.store, toks, "dynamic", plan=plan)
    bits_d, _ = trace_arrays(tr.steps, ids)
    s_end = len(bits_d)
    for s in range(len(bits_d)):
        if not np.array_equal(bits_d[s], golden_traces["linear_bits"][s]):
            s_end = s + 1
            break
    assert not decision_mismatches(bits_d[:s_end], golden_traces["linear_bits"][:s_end],
                                   golden_traces["linear_est"][:s_end], Ts(plan, ids), EPS_DECISION["f32"])


def test_fp_mode(report_setup, golden_summary):
    losses = []
    for toks in report_setup.chunks:
        _, tr = R.eval_perplexity(report_setup.weights, report_setup.store, toks, "fp")
        losses.extend(tr.token_losses)
    assert float(np.exp(np.mean(losses))) == pytest.approx(golden_summary["fp_perplexity"], rel=1e-10)


def _mixed_bits(store):
    return {lid: (4 if lid.kind in ("q", "k", "v") else 5) for lid in store.layers}


def test_stepwise_matches_batch_forward(toy_weights, toy_store):
    bits = _mixed_bits(toy_store)
    toks = np.random.default_rng(0).integers(0, 256, 30)
    layers = {O.key(l): O.as_layer(q) for l, q in toy_store.layers.items()}
    mats = {k: O.dequantize(layers[k], bits[M.LayerId(*k)]) for k in layers}
    logits = O.forward(toy_weights.config, toy_weights.embed, toy_weights.lm_head, lambda k: mats[k], toks)
    ref = O.token_losses(logits, toks)
    from paper_2508_06041_b200.runtime import sentinel_static_plan
    asg = type("A", (), {"bits": bits})()
    ppl, tr = R.eval_perplexity(toy_weights, toy_store, toks, "static", assignment=asg)
    np.testing.assert_allclose(tr.token_losses, ref, atol=LOSS_TOL)
    assert ppl == pytest.approx(float(np.exp(ref.mean())), rel=1e-5)


def test_sentinel_dynamic_equals_static_exactly(toy_weights, toy_store):
    bits = _mixed_bits(toy_store)
    toks = np.arange(25)
    asg = type("A", (), {"bits": bits})()
    ppl_s, tr_s = R.eval_perplexity(toy_weights, toy_store, toks, "static", assignment=asg)
    plan = R.sentinel_static_plan(bits, toy_store.param_counts(), 4.5)
    ppl_d, tr_d = R.eval_perplexity(toy_weights, toy_store, toks, "dynamic", plan=plan)
    assert ppl_d == ppl_s
    assert tr_d.token_losses == tr_s.token_losses
    assert [s.bits for s in tr_d.steps] == [s.bits for s in tr_s.steps]


def test_forced_static_equivalence_c8(toy_weights, toy_store):
    """Acceptance C8 (tests/test_acceptance.py:234-272): +inf on (a, a+1) and
    -inf on (a-1, a) reproduce the static assignment exactly, device vs device."""
    rng = np.random.default_rng(8)
    bits = {lid: int(rng.integers(3, 7)) for lid in toy_store.layers}
    counts = toy_store.param_counts()
    toks = rng.integers(0, 256, 20)
    asg = type("A", (), {"bits": bits})()
    ppl_s, tr_s = R.eval_perplexity(toy_weights, toy_store, toks, "static", assignment=asg)
    lo = {lid: R.PlanLayer(lid, a, float(a), (a, min(a + 1, 6)), np.inf, 1.0, None) for lid, a in bits.items()}
    hi = {lid: R.PlanLayer(lid, a, float(a), (max(a - 1, 3), a), -np.inf, 0.0, None) for lid, a in bits.items()}
    for layers in (lo, hi):
        plan = R.PrecisionPlan("x", 4.0, float("nan"), layers, counts)
        ppl_f, tr_f = R.eval_perplexity(toy_weights, toy_store, toks, "dynamic", plan=plan)
        assert ppl_f == ppl_s and tr_f.token_losses == tr_s.token_losses
        assert all(s.bits[lid] == bits[lid] for s in tr_f.steps for lid in s.bits)
    out_s, _ = R.decode(toy_weights, toy_store, R.sentinel_static_plan(bits, counts, 4.0), toks[:6], 8)
    out_f, _ = R.decode(toy_weights, toy_store, R.PrecisionPlan("x", 4.0, float("nan"), lo, counts),
                        toks[:6], 8)
    assert out_s == out_f


def test_effective_bits_and_trace_csv(tmp_path, toy_weights, toy_store):
    plan = R.sentinel_static_plan({l: 4 for l in toy_store.layers}, toy_store.param_counts(), 4.0)
    _, tr = R.eval_perplexity(toy_weights, toy_store, np.arange(10), "dynamic", plan=plan)
    assert np.isclose(tr.mean_effective_bits(), 4.0)
    p = str(tmp_path / "t.csv")
    tr.export_csv(p)
    lines = open(p).read().splitlines()
    assert lines[0] == "step,layer,bit,estimate"
    assert len(lines) == 1 + len(tr.steps) * len(plan.layers)


def test_greedy_deterministic_and_cap(toy_weights, toy_store):
    plan = R.sentinel_static_plan({l: 4 for l in toy_store.layers}, toy_store.param_counts(), 4.0)
    a, tr = R.decode(toy_weights, toy_store, plan, np.arange(5), 12)
    b, _ = R.decode(toy_weights, toy_store, plan, np.arange(5), 12)
    assert a == b and len(a) == 12 and len(tr.steps) == 12
    eng = R.DecodeEngine(toy_weights, toy_store, plan)
    for t in range(toy_weights.config.seq_cap):
        eng.step(t % 256, dynamic=False, want_logits=False)
    with pytest.raises(ValueError):
        eng.step(0)


def synthetic_projection_plan(store, pairs, k=16, seed=0, T_scale=None):
    """Projection plan with G = A dW (oracle float64) and T picked per layer."""
    layers, Ms = {}, store.param_counts()
    rng = np.random.default_rng(seed)
    for i, lid in enumerate(canon(store.layers)):
        q = O.as_layer(store.layers[lid])
        l, h = pairs[lid]
        A = rng.standard_normal((k, q.shape[0])) / np.sqrt(k)
        G = A @ O.delta_weights(q, l, h)
        est = R.E.ErrorEstimator(R.E.ProjectionEstimator(G, k, seed), R.E.IMMEDIATE, (l, h))
        layers[lid] = R.PlanLayer(lid, h, l + 0.5, (l, h), 1.0, 0.5, est)
    return R.PrecisionPlan("dp", 3.5, 4.0, layers, Ms)


def calibrate_T(weights, store, plan, tokens, q=0.5):
    """T := per-layer quantile of the oracle's estimates over a calibration run."""
    for pl in plan.layers.values():
        pl.T = 1e300
    _, _, eng = oracle_eval(weights, store, plan, tokens)
    for lid, pl in plan.layers.items():
        vals = np.sort([r.estimates[O.key(lid)] for r in eng.records])
        pl.T = float(vals[int(q * (len(vals) - 1))])
    return plan


@pytest.mark.parametrize("gqa", [False, True])
def test_cfg1_model_forced_and_free(gqa):
    """cfg1 shapes (2 blocks, d=512, d_ff=1792, 4/3-bit store) and a GQA
    variant: logits vs the oracle under forced replay; free-run decisions."""
    cfg = M.ModelConfig(n_blocks=2, d_model=512, n_heads=8, d_ff=1792, vocab=256, seq_cap=64,
                        n_kv_heads=2 if gqa else None)
    w = M.init_model(0, cfg)
    store = Q.quantize_model(w, 4, 3)
    plan = synthetic_projection_plan(store, {l: (3, 4) for l in store.layers}, k=64)
    toks = np.random.default_rng(3).integers(0, 256, 24)
    calibrate_T(w, store, plan, toks[:12])
    ids = canon(store.layers)
    _, ls_o, eng_o = oracle_eval(w, store, plan, toks)
    forced = forced_from_oracle(eng_o, ids)
    ls, eng, lg = device_eval_forced(w, store, plan, toks, forced, g_dtype="f32")
    np.testing.assert_allclose(ls, ls_o, atol=LOSS_TOL)
    bits_o, est_o = trace_arrays(eng_o.records, ids)
    _, est_d = trace_arrays(eng.trace.steps, ids)
    np.testing.assert_allclose(est_d, est_o, rtol=1e-4)
    # free run with f16 G: decisions until the first eps-tie
    _, tr = R.eval_perplexity(w, store, toks, "dynamic", plan=plan)
    bits_d, _ = trace_arrays(tr.steps, ids)
    for s in range(len(bits_o)):
        assert not decision_mismatches(bits_d[s:s + 1], bits_o[s:s + 1], est_o[s:s + 1], Ts(plan, ids),
                                       EPS_DECISION["f16"])
        if not np.array_equal(bits_d[s], bits_o[s]):
            break


def test_async_prev_step_and_prev_block_projection(toy_weights, toy_store):
    """Previous-residual projection estimators through the snapshot path."""
    plan = synthetic_projection_plan(toy_store, {l: (3, 4) for l in toy_store.layers}, k=8, seed=2)
    for lid, pl in plan.layers.items():
        if lid.residual_fed and lid.block > 0:
            pl.estimator.input_source = R.E.PREVIOUS_RESIDUAL
    toks = np.random.default_rng(5).integers(0, 256, 20)
    calibrate_T(toy_weights, toy_store, plan, toks[:10])
    ids = canon(toy_store.layers)
    for rule in ("prev_step", "prev_block"):
        for prime in (True, False):
            _, ls_o, eng_o = oracle_eval(toy_weights, toy_store, plan, toks, async_rule=rule,
                                         prime_from_prefill=prime)
            forced = forced_from_oracle(eng_o, ids)
            ls, eng, _ = device_eval_forced(toy_weights, toy_store, plan, toks, forced, async_rule=rule,
                                            prime_from_prefill=prime, g_dtype="f32")
            np.testing.assert_allclose(ls, ls_o, atol=LOSS_TOL)
            _, est_o = trace_arrays(eng_o.records, ids)
            _, est_d = trace_arrays(eng.trace.steps, ids)
            np.testing.assert_allclose(est_d, est_o, rtol=1e-4)


@pytest.mark.parametrize("gqa", [False, True])
def test_engine_matches_multi_kernel_and_is_deterministic(gqa):
    """The persistent engine (producer-fused estimators, fixed-point
    accumulation) and the per-op kernel graph agree under forced-bits replay;
    two engine runs are bit-identical (logits, decisions, estimates)."""
    cfg = M.ModelConfig(n_blocks=3, d_model=256, n_heads=8, d_ff=768, vocab=256, seq_cap=160,
                        n_kv_heads=2 if gqa else None)
    w = M.init_model(1, cfg)
    store = Q.quantize_model(w, 5, 3)
    plan = synthetic_projection_plan(store, {l: (3, 4) for l in store.layers}, k=32, seed=4)
    toks = np.random.default_rng(9).integers(0, 256, 90)
    calibrate_T(w, store, plan, toks[:12])
    ids = store.ordered_ids()
    runs = []
    for _ in range(2):
        eng = R.DecodeEngine(w, store, plan)
        assert eng.persistent
        lg = [eng.step(int(toks[0]), dynamic=False)]
        for t in toks[1:]:
            lg.append(eng.step(int(t), dynamic=True))
        runs.append((np.array(lg), [s.bits for s in eng.trace.steps],
                     [s.estimates for s in eng.trace.steps]))
    assert np.array_equal(runs[0][0], runs[1][0])
    assert runs[0][1] == runs[1][1]
    assert runs[0][2] == runs[1][2]
    old = R.DecodeEngine(w, store, plan, use_persistent=False)
    assert not old.persistent
    lg = [old.step(int(toks[0]), dynamic=False)]
    for t, bits in zip(toks[1:], runs[0][1]):
        lg.append(old.step(int(t), dynamic=True, forced_bits=bits))
    lg = np.array(lg)
    assert np.max(np.abs(lg - runs[0][0])) <= 1e-4 * np.max(np.abs(lg))
    est_e = np.array([[e[l] for l in ids] for e in runs[0][2]])
    est_o = np.array([[s.estimates[l] for l in ids] for s in old.trace.steps])
    np.testing.assert_allclose(est_e, est_o, rtol=1e-4)
    T = np.array([plan.layers[l].T for l in ids])
    hi = np.array([plan.layers[l].pair[1] for l in ids])
    lo = np.array([plan.layers[l].pair[0] for l in ids])
    want = np.where(est_o > T, hi, lo)
    got = np.array([[b[l] for l in ids] for b in runs[0][1]])
    near = np.abs(est_o - T) <= 1e-3 * np.abs(T)
    assert np.all((got == want) | near)


@pytest.mark.gpu
@pytest.mark.parametrize("width", ["llama3_8b", "llama2_7b", "llama2_70b"])
def test_engine_llama_width_two_blocks(width):
    """The engine at the bench's layer widths (8B: d 4096, 32 heads / 8 KV,
    d_ff 14336, 8 and 28 column windows; 70B: d 8192, 64 heads / 8 KV, d_ff
    28672, 16 and 56 windows, a 6-bit overlay with mixed (3,4) / (4,5) pairs;
    window-aligned CTA split, several runs per CTA, extra planes across
    windows; at 70B widths a CTA owns up to ~270 groups of up|gate, so parked
    base sums overflow the shared table into the global scratch) against the
    per-op kernel graph under forced-bits replay, and bit-identical across
    runs."""
    import paper_2508_06041_b200.synth as S
    if width == "llama3_8b":
        cfg = M.ModelConfig(n_blocks=2, d_model=4096, n_heads=32, d_ff=14336, vocab=256, seq_cap=64,
                            n_kv_heads=8)
        n_bits = 4
    elif width == "llama2_7b":             # MHA; d_ff 11008 = 21.5 windows (ragged last window)
        cfg = M.ModelConfig(n_blocks=2, d_model=4096, n_heads=32, d_ff=11008, vocab=256, seq_cap=64)
        n_bits = 4
    else:
        cfg = M.ModelConfig(n_blocks=1, d_model=8192, n_heads=64, d_ff=28672, vocab=256, seq_cap=64,
                            n_kv_heads=8)
        n_bits = 6
    w, store, _ = S.random_device_model(cfg, n_bits, 3, seed=77)
    ids = store.ordered_ids()
    pairs = {l: ((3, 4) if n_bits == 4 or i % 2 == 0 else (4, 5)) for i, l in enumerate(ids)}
    plan = S.projection_plan(store, pairs, {l: pairs[l][1] for l in ids}, k=64, seed=3, target=3.5)
    toks = np.random.default_rng(12).integers(0, 256, 14)
    S.calibrate_thresholds(w, store, plan, toks[:6], high_rate=0.5)
    runs = []
    for _ in range(2):
        eng = R.DecodeEngine(w, store, plan)
        from paper_2508_06041_b200 import _lib
        assert _lib.load().dpq_session_is_persistent(eng._h) == 2      # the TMA engine
        lg = [eng.step(int(toks[0]), dynamic=False)]
        for t in toks[1:]:
            lg.append(eng.step(int(t), dynamic=True))
        runs.append((np.array(lg), [s.bits for s in eng.trace.steps]))
        eng.close()
    assert np.array_equal(runs[0][0], runs[1][0]) and runs[0][1] == runs[1][1]
    highs = np.mean([[b[l] == pairs[l][1] for l in ids] for b in runs[0][1]])
    assert 0.05 < highs < 0.95                    # both precisions exercised
    old = R.DecodeEngine(w, store, plan, use_persistent=False)
    lg = [old.step(int(toks[0]), dynamic=False)]
    for t, bits in zip(toks[1:], runs[0][1]):
        lg.append(old.step(int(t), dynamic=True, forced_bits=bits))
    lg = np.array(lg)
    assert np.max(np.abs(lg - runs[0][0])) <= 1e-4 * np.max(np.abs(lg))
    assert np.array_equal(np.argmax(lg, axis=1), np.argmax(runs[0][0], axis=1))


@pytest.mark.gpu
@pytest.mark.parametrize("d_model,n_heads", [(128, 4), (64, 4)])
def test_engine_long_context_chunked_attention(d_model, n_heads):
    """Past one attention unit (15 warps x 16 positions = 240) the engine splits
    a head's positions into chunks merged by the last unit; head_dim 32 emits
    per head, head_dim 16 goes through the EMIT stage. Compared with the per-op
    kernel graph under forced-bits replay."""
    cfg = M.ModelConfig(n_blocks=1, d_model=d_model, n_heads=n_heads, d_ff=2 * d_model, vocab=256,
                        seq_cap=320)
    w = M.init_model(5, cfg)
    store = Q.quantize_model(w, 5, 3)
    plan = synthetic_projection_plan(store, {l: (3, 4) for l in store.layers}, k=16, seed=8)
    toks = np.random.default_rng(13).integers(0, 256, 300)
    calibrate_T(w, store, plan, toks[:10])
    eng = R.DecodeEngine(w, store, plan)
    assert eng.persistent
    lg = [eng.step(int(toks[0]), dynamic=False)]
    for t in toks[1:]:
        lg.append(eng.step(int(t), dynamic=True))
    bits = [s.bits for s in eng.trace.steps]
    old = R.DecodeEngine(w, store, plan, use_persistent=False)
    lo = [old.step(int(toks[0]), dynamic=False)]
    for t, b in zip(toks[1:], bits):
        lo.append(old.step(int(t), dynamic=True, forced_bits=b))
    lg, lo = np.array(lg), np.array(lo)
    assert np.max(np.abs(lg - lo)) <= 1e-4 * np.max(np.abs(lo))
    assert np.max(np.abs(lg[250:] - lo[250:])) <= 1e-4 * np.max(np.abs(lo))   # the chunked positions


def test_trace_pulled_lazily_keeps_positions(report_setup):
    """The trace is pulled from the device on access (not per step): records
    keep the positions of the dynamic steps, also around non-dynamic steps and
    device-loop launches, and mid-run reads do not change the result."""
    S = report_setup
    plan = R.load_plan(plan_path("dp_t3.5"), S.store)
    prompt = S.tokens[:4]

    def run(peek):
        eng = R.DecodeEngine(S.weights, S.store, plan, S.store_hash)
        eng.prefill(prompt)
        for t in S.tokens[4:7]:
            eng.step(int(t), dynamic=True, want_logits=False)
            if peek:
                assert len(eng.trace.steps) == eng.position - len(prompt)
        eng.step(int(S.tokens[7]), dynamic=False, want_logits=False)
        eng.decode_greedy(2)
        return eng.trace

    a, b = run(True), run(False)
    assert [s.step for s in a.steps] == [4, 5, 6, 8, 9]
    assert [s.step for s in b.steps] == [4, 5, 6, 8, 9]
    assert [s.bits for s in a.steps] == [s.bits for s in b.steps]
    assert a.estimator_ops == b.estimator_ops > 0


@pytest.mark.parametrize("kind", ["flag_kernel", "per_op_graph"])
def test_non_engine_session_kinds_match_oracle(monkeypatch, kind):
    """The decode paths used when the TMA engine declines a shape
    (DPQ_ENGINE=0 here): the persistent flag-linked step_kernel (session kind
    1) and the multi-kernel op graph (kind 0). Logits vs the oracle under
    forced replay, free-run decisions under the eps rule."""
    from paper_2508_06041_b200 import _lib
    monkeypatch.setenv("DPQ_ENGINE", "0")
    cfg = M.ModelConfig(n_blocks=2, d_model=256, n_heads=4, d_ff=512, vocab=256, seq_cap=64, n_kv_heads=2)
    w = M.init_model(5, cfg)
    store = Q.quantize_model(w, 5, 3)
    plan = synthetic_projection_plan(store, {l: (3, 4) for l in store.layers}, k=32, seed=2)
    toks = np.random.default_rng(3).integers(0, 256, 16)
    calibrate_T(w, store, plan, toks[:8])
    ids = canon(store.layers)
    eng = R.DecodeEngine(w, store, plan, g_dtype="f32", use_persistent=(kind == "flag_kernel"))
    assert _lib.load().dpq_session_is_persistent(eng._h) == (1 if kind == "flag_kernel" else 0)
    lg = [eng.step(int(toks[0]), dynamic=False)] + [eng.step(int(t)) for t in toks[1:]]
    bits_d, _ = trace_arrays(eng.trace.steps, ids)
    eo = oracle_engine(w, store, plan)
    ref_free = [eo.step(int(toks[0]), dynamic=False)] + [eo.step(int(t)) for t in toks[1:]]
    bits_o, est_o = trace_arrays(eo.records, ids)
    assert not decision_mismatches(bits_d, bits_o, est_o, Ts(plan, ids), EPS_DECISION["f32"])
    eo2 = oracle_engine(w, store, plan)
    eo2.forced = [{O.key(l): int(b) for l, b in zip(ids, row)} for row in bits_d]
    ref = [eo2.step(int(toks[0]), dynamic=False)] + [eo2.step(int(t)) for t in toks[1:]]
    assert np.max(np.abs(np.array(lg) - np.array(ref))) <= LOGIT_TOL * np.max(np.abs(ref))
    eng.close()


def test_engine_e4m3_projection():
    """fp8-e4m3 G (per-row scale) on the TMA engine: estimates within the e4m3
    rounding of the oracle's, decisions under the e4m3 eps rule."""
    from paper_2508_06041_b200 import _lib
    cfg = M.ModelConfig(n_blocks=2, d_model=256, n_heads=4, d_ff=512, vocab=256, seq_cap=64, n_kv_heads=2)
    w = M.init_model(6, cfg)
    store = Q.quantize_model(w, 5, 3)
    plan = synthetic_projection_plan(store, {l: (3, 4) for l in store.layers}, k=32, seed=4)
    toks = np.random.default_rng(5).integers(0, 256, 16)
    calibrate_T(w, store, plan, toks[:8])
    ids = canon(store.layers)
    eng = R.DecodeEngine(w, store, plan, g_dtype="e4m3")
    assert _lib.load().dpq_session_is_persistent(eng._h) == 2
    eo = oracle_engine(w, store, plan)
    bits_o = []
    eng.step(int(toks[0]), dynamic=False)
    eo.step(int(toks[0]), dynamic=False)
    for t in toks[1:]:
        eo.step(int(t))
        row = np.array([eo.records[-1].bits[O.key(l)] for l in ids], dtype=np.int8)
        eng.step(int(t), forced_bits=row)             # same inputs: compare the estimates
        bits_o.append(row)
    _, est_d = trace_arrays(eng.trace.steps, ids)
    _, est_o = trace_arrays(eo.records, ids)
    np.testing.assert_allclose(est_d, est_o, rtol=3e-2)
    eng.close()


def _dual_setup(kind):
    cfg = M.ModelConfig(n_blocks=2, d_model=256, n_heads=4, d_ff=512, vocab=256, seq_cap=64, n_kv_heads=2)
    w = M.init_model(9, cfg)
    store = Q.quantize_model(w, 5, 3)
    pairs = {l: (3, 4) for l in store.layers}
    if kind == "projection":
        plan = synthetic_projection_plan(store, pairs, k=32, seed=3)
    else:
        layers = {}
        for lid in store.layers:
            est = R.E.ErrorEstimator(R.E.ExactEstimator(store.layers[lid], 3, 4), R.E.IMMEDIATE, (3, 4))
            layers[lid] = R.PlanLayer(lid, 4, 3.5, (3, 4), 1.0, 0.5, est)
        plan = R.PrecisionPlan("dp", 3.5, 4.0, layers, store.param_counts())
    toks = np.random.default_rng(21).integers(0, 256, 16)
    calibrate_T(w, store, plan, toks[:8])
    return w, store, plan, toks


@pytest.mark.parametrize("kind", ["projection", "exact"])
def test_engine_dual_layers_match_oracle(kind):
    """Exact estimators (estimator.py:63-73, decision from ||(W_h - W_l) x||)
    and track_exact (runtime.py:322-324) on the TMA engine (dual units: all h
    planes, y_l and y_h from the shared planes): forced replay of the
    oracle's decisions gives its logits, estimates and exact errors; the free
    run's decisions follow the oracle under the eps rule."""
    from paper_2508_06041_b200 import _lib
    w, store, plan, toks = _dual_setup(kind)
    ids = canon(store.layers)
    eo = oracle_engine(w, store, plan, track_exact=True)
    ref = [eo.step(int(toks[0]), dynamic=False)] + [eo.step(int(t)) for t in toks[1:]]
    bits_o, est_o = trace_arrays(eo.records, ids)
    xerr_o = np.array([[r.exact_errors[O.key(l)] for l in ids] for r in eo.records])
    eng = R.DecodeEngine(w, store, plan, g_dtype="f32", track_exact=True)
    assert _lib.load().dpq_session_is_persistent(eng._h) == 2, "not on the TMA engine"
    lg = [eng.step(int(toks[0]), dynamic=False)]
    for i, t in enumerate(toks[1:]):
        lg.append(eng.step(int(t), forced_bits=bits_o[i].astype(np.int8)))
    lg = np.array(lg)
    assert np.max(np.abs(lg - np.array(ref))) <= LOGIT_TOL * np.max(np.abs(ref))
    bits_d, est_d = trace_arrays(eng.trace.steps, ids)
    np.testing.assert_array_equal(bits_d, bits_o)
    np.testing.assert_allclose(est_d, est_o, rtol=1e-4, atol=1e-9)
    xerr_d = np.array([[s.exact_errors[l] for l in ids] for s in eng.trace.steps])
    np.testing.assert_allclose(xerr_d, xerr_o, rtol=1e-4, atol=1e-9)
    eng.close()
    # free run: the device's own decisions
    eng = R.DecodeEngine(w, store, plan, g_dtype="f32", track_exact=True)
    eng.step(int(toks[0]), dynamic=False)
    for t in toks[1:]:
        eng.step(int(t))
    bits_f, _ = trace_arrays(eng.trace.steps, ids)
    assert not decision_mismatches(bits_f, bits_o, est_o, Ts(plan, ids), EPS_DECISION["f32"])
    assert 0.1 < np.mean(bits_f == 4) < 0.9
    eng.close()
