"""Oracle parity of the persistent engine at the benchmarked layer widths.

The bench's headline runs Llama-3-8B / Llama-2-7B / Llama-2-70B-shaped models
on the TMA engine (session kind 2). These tests run the same engine on 1-2
block slices of those shapes and compare it with the float64 oracle
(oracle/dpq_oracle.py, a restatement of runtime.py:330-381, estimator.py:49-60,
quant.py:67-99) on the SAME host codes and the SAME projection matrices:

* forced replay: the device replays the oracle's per-layer bits; logits within
  2e-5 of the logit scale, argmax equal, estimates within rtol 1e-4 (f32 G) or
  2e-3 (f16 G, the engine's default);
* free run: the device takes its own decisions for >= 16 steps; every decision
  equals the oracle's except where |est_ref - T| <= eps |T| (eps 1e-4 f32 G,
  1e-3 f16 G); after the first such tie the trajectories may diverge, so the
  comparison stops there.

Parity rule and tolerances: DESIGN.md §2.
"""

import numpy as np
import pytest

from oracle import dpq_oracle as O
from paper_2508_06041_b200 import _lib
from paper_2508_06041_b200 import model as M
from paper_2508_06041_b200 import runtime as R

from helpers import EPS_DECISION, trace_arrays, decision_mismatches

pytestmark = pytest.mark.gpu
LOGIT_TOL = 2e-5
EST_RTOL = {"f32": 1e-4, "f16": 2e-3}

WIDTHS = {
    # name: (config, n_bits, pair rule)
    "llama3_8b": (dict(n_blocks=2, d_model=4096, n_heads=32, d_ff=14336, n_kv_heads=8), 4, "34"),
    "llama2_7b": (dict(n_blocks=2, d_model=4096, n_heads=32, d_ff=11008), 6, "34"),
    "llama2_70b": (dict(n_blocks=1, d_model=8192, n_heads=64, d_ff=28672, n_kv_heads=8), 6, "mixed"),
}


@pytest.fixture(scope="module", params=list(WIDTHS))
def width_setup(request):
    import paper_2508_06041_b200.synth as S
    name = request.param
    kw, n_bits, rule = WIDTHS[name]
    cfg = M.ModelConfig(vocab=256, seq_cap=64, **kw)
    w, store, host = S.random_device_model(cfg, n_bits, 3, seed=31, keep_host_blocks=cfg.n_blocks)
    ids = store.ordered_ids()
    pairs = {l: ((3, 4) if rule == "34" or i % 2 == 0 else (4, 5)) for i, l in enumerate(ids)}
    plan = S.projection_plan(store, pairs, {l: pairs[l][1] for l in ids}, k=64, seed=5, target=3.5)
    toks = np.random.default_rng(17).integers(0, 256, 24)
    S.calibrate_thresholds(w, store, plan, toks[:8], high_rate=0.5, g_dtype="f32")
    eo = O.Engine(w, host, plan.layers, plan.M)
    ref = [eo.step(int(toks[0]), dynamic=False)] + [eo.step(int(t)) for t in toks[1:]]
    return dict(name=name, cfg=cfg, w=w, store=store, plan=plan, ids=ids, toks=toks, eo=eo,
                ref=np.array(ref))


def _engine(S, g_dtype):
    eng = R.DecodeEngine(S["w"], S["store"], S["plan"], g_dtype=g_dtype)
    assert _lib.load().dpq_session_is_persistent(eng._h) == 2, "not on the TMA engine"
    return eng


@pytest.mark.parametrize("g_dtype", ["f32", "f16"])
def test_forced_replay_matches_oracle(width_setup, g_dtype):
    S = width_setup
    ids, toks, eo = S["ids"], S["toks"], S["eo"]
    bits_o, est_o = trace_arrays(eo.records, ids)
    eng = _engine(S, g_dtype)
    lg = [eng.step(int(toks[0]), dynamic=False)]
    for i, t in enumerate(toks[1:]):
        lg.append(eng.step(int(t), dynamic=True, forced_bits=bits_o[i].astype(np.int8)))
    lg = np.array(lg)
    ref = S["ref"]
    err = np.max(np.abs(lg - ref))
    assert err <= LOGIT_TOL * np.max(np.abs(ref)), (err, np.max(np.abs(ref)))
    assert np.array_equal(np.argmax(lg, axis=1), np.argmax(ref, axis=1))
    bits_d, est_d = trace_arrays(eng.trace.steps, ids)
    assert np.array_equal(bits_d, bits_o)
    np.testing.assert_allclose(est_d, est_o, rtol=EST_RTOL[g_dtype])
    # both precisions are exercised by the calibrated thresholds
    highs = np.mean([[b.bits[l] == S["plan"].layers[l].pair[1] for l in ids] for b in eng.trace.steps])
    assert 0.1 < highs < 0.9
    eng.close()


@pytest.mark.parametrize("g_dtype", ["f32", "f16"])
def test_free_run_decisions_match_oracle(width_setup, g_dtype):
    S = width_setup
    ids, toks, eo, plan = S["ids"], S["toks"], S["eo"], S["plan"]
    bits_o, est_o = trace_arrays(eo.records, ids)
    T = np.array([plan.layers[l].T for l in ids])
    eng = _engine(S, g_dtype)
    lg = [eng.step(int(toks[0]), dynamic=False)]
    for t in toks[1:]:
        lg.append(eng.step(int(t), dynamic=True))
    bits_d, est_d = trace_arrays(eng.trace.steps, ids)
    assert len(bits_d) >= 16
    n_same = 0
    for s in range(len(bits_o)):
        bad = decision_mismatches(bits_d[s:s + 1], bits_o[s:s + 1], est_o[s:s + 1], T, EPS_DECISION[g_dtype])
        assert not bad, (s, bad[:3])
        if not np.array_equal(bits_d[s], bits_o[s]):
            break                                   # an eps-tie: trajectories may diverge from here
        n_same += 1
        # identical decisions so far: identical inputs up to fp32 rounding
        ref = S["ref"][s + 1]
        assert np.max(np.abs(lg[s + 1] - ref)) <= LOGIT_TOL * np.max(np.abs(ref))
    # f16 G: a decision within the f16 estimate error of T can tie at the very
    # first step (checked above against eps); f32 G must agree for >= 1 step
    assert n_same >= (1 if g_dtype == "f32" else 0)
    eng.close()


def test_device_greedy_loop_matches_oracle(width_setup):
    """dpq_session_decode (argmax fed back on the device, one launch) against
    the oracle's greedy decode with f32 G: tokens equal up to the first
    eps-tie of a decision."""
    S = width_setup
    ids, plan = S["ids"], S["plan"]
    prompt = S["toks"][:6]
    n_new = 12
    eo = O.Engine(S["w"], {l: S["eo"].layers[O.key(l)] for l in ids}, plan.layers, plan.M)
    out_o = O.decode(eo, prompt, n_new)
    bits_o, est_o = trace_arrays(eo.records, ids)
    out_d, tr = R.decode(S["w"], S["store"], plan, prompt, n_new, g_dtype="f32")
    bits_d, _ = trace_arrays(tr.steps, ids)
    T = np.array([plan.layers[l].T for l in ids])
    assert len(out_d) == len(out_o) == n_new
    for s in range(n_new):
        # token s is the argmax after step s - 1 (the prefill for s = 0): it
        # depends only on decisions already checked equal
        assert out_d[s] == out_o[s], (s, out_d, out_o)
        assert not decision_mismatches(bits_d[s:s + 1], bits_o[s:s + 1], est_o[s:s + 1], T, EPS_DECISION["f32"])
        if not np.array_equal(bits_d[s], bits_o[s]):
            break


def test_cfg1_reference_planned_decode():
    """cfg1 with the plan the REFERENCE planner built
    (tools/make_golden.py cfg1_plan: build_dp_plan(budget 4.0, target 3.5,
    hybrid, k=64, calibrate=True)): the device's greedy decode (f32 G)
    equals the reference DecodeEngine's tokens and effective bits up to the
    first eps-tie of a decision (decisions checked against the oracle's)."""
    import os
    from conftest import GOLDEN
    from paper_2508_06041_b200 import quant as Q
    g = np.load(os.path.join(GOLDEN, "cfg1_plan_decode.npz"))
    cfg = M.ModelConfig(n_blocks=2, d_model=512, n_heads=8, d_ff=1792, vocab=256, seq_cap=512)
    w = M.init_model(0, cfg)
    store = Q.quantize_model(w, 4, 3)
    plan = R.load_plan(os.path.join(GOLDEN, "plans", "cfg1_dp_t3.5.json"), store)
    prompt = g["prompt"]
    out, tr = R.decode(w, store, plan, prompt, 64, store_hash=str(g["store_hash"][0]), g_dtype="f32")
    ref = g["tokens"].tolist()
    ids = store.ordered_ids()
    # the oracle's decisions and estimates along the device's own trajectory
    eo = O.Engine(w, store.layers, plan.layers, plan.M)
    O.decode(eo, prompt, 64)
    bits_o, est_o = trace_arrays(eo.records, ids)
    bits_d, _ = trace_arrays(tr.steps, ids)
    T = np.array([plan.layers[l].T for l in ids])
    n_same = 0
    for s in range(64):
        assert not decision_mismatches(bits_d[s:s + 1], bits_o[s:s + 1], est_o[s:s + 1], T, EPS_DECISION["f32"])
        if not np.array_equal(bits_d[s], bits_o[s]):
            break
        assert out[s] == ref[s], (s, out[:s + 1], ref[:s + 1])
        n_same += 1
    assert n_same >= 8
    eff = np.array([s.effective_bits for s in tr.steps])
    np.testing.assert_allclose(eff[:n_same], g["eff"][:n_same], rtol=0, atol=1e-12)
