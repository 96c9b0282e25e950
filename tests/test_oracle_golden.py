"""Pin the CPU oracle (oracle/dpq_oracle.py) against vectors produced by the
unmodified reference (tools/make_golden.py). CPU only."""

import numpy as np
import pytest

from oracle import dpq_oracle as O
from paper_2508_06041_b200 import model as M
from paper_2508_06041_b200 import runtime as R

from conftest import plan_path
from helpers import canon, oracle_engine, oracle_eval, trace_arrays


def test_kat_two_bit(quant_vectors):
    q = O.quantize_layer(np.array([[0.0, 0.3, 0.6, 1.0]]), 2, 2)
    assert q.codes.tolist() == quant_vectors["kat2_codes"].tolist() == [[0, 1, 2, 3]]
    assert np.array_equal(O.dequantize(q, 2), quant_vectors["kat2_deq"])


@pytest.mark.parametrize("case", range(6))
def test_quant_vectors(quant_vectors, case):
    g = quant_vectors
    r, c, n, bmin = (int(v) for v in g[f"c{case}_meta"])
    codes, lo, hi = g[f"c{case}_codes"], g[f"c{case}_lo"], g[f"c{case}_hi"]
    if f"c{case}_W" in g:
        q = O.quantize_layer(g[f"c{case}_W"], n, bmin)
        assert np.array_equal(q.codes, codes)
        assert np.array_equal(q.lo, lo) and np.array_equal(q.hi, hi)
    q = O.Layer(codes, n, bmin, lo, hi)
    x = g[f"c{case}_x"]
    for b in range(bmin, n + 1):
        if g[f"c{case}_deq{b}"].size:
            assert np.array_equal(O.dequantize(q, b), g[f"c{case}_deq{b}"])
        y_ref = g[f"c{case}_y{b}"]
        np.testing.assert_allclose(O.gemv(q, b, x), y_ref, rtol=1e-12, atol=1e-12)
        # the plane-sum algebra the kernel implements
        np.testing.assert_allclose(O.plane_sum_gemv(q, b, x), y_ref, rtol=1e-10,
                                   atol=1e-10 * np.abs(y_ref).max())
    if n > bmin:
        np.testing.assert_allclose(O.exact_error(q, bmin, bmin + 1, x), g[f"c{case}_exact"][0],
                                   rtol=1e-12)
    assert O.pack_codes(codes, n) == g[f"c{case}_packed"].tobytes()
    assert np.array_equal(O.unpack_codes(g[f"c{case}_packed"].tobytes(), n, codes.shape), codes)


def test_nesting_prefix_and_mse():
    # reference tests/test_acceptance.py:28-43 on the oracle
    rng = np.random.default_rng(10)
    for _ in range(10):
        W = rng.normal(size=(int(rng.integers(1, 64)), int(rng.integers(1, 64))))
        q = O.quantize_layer(W, 6, 3)
        prev = np.inf
        for b in (3, 4, 5, 6):
            if b < 6:
                assert np.array_equal(q.codes >> (6 - b), (q.codes >> (5 - b)) >> 1)
            mse = float(np.mean((O.dequantize(q, b) - W) ** 2))
            assert mse <= prev
            prev = mse


def test_fp_perplexity(report_setup, golden_summary):
    losses = []
    for toks in report_setup.chunks:
        _, per = O.fp_perplexity(report_setup.weights, toks)
        losses.extend(per)
    ppl = float(np.exp(np.mean(losses)))
    assert ppl == pytest.approx(golden_summary["fp_perplexity"], rel=1e-12)


@pytest.mark.parametrize("name", ["dp_t3.5", "dp_t4", "llm_mq_t3.5", "hawq_v2_t4"])
def test_shipped_plans_report_numbers(report_setup, golden_summary, golden_traces, name):
    """report.csv rows (artifacts/reports/report.csv:3-12) from the oracle."""
    S = report_setup
    plan = R.load_plan(plan_path(name), S.store)
    losses, effs, ops = [], [], 0
    first = None
    for ci, toks in enumerate(S.chunks):
        _, ls, eng = oracle_eval(S.weights, S.store, plan, toks)
        losses.extend(ls)
        effs.append(np.mean([r.effective_bits for r in eng.records]))
        ops += eng.estimator_ops
        if ci == 0:
            first = eng
    exp = golden_summary["plans"][name]
    assert float(np.exp(np.mean(losses))) == pytest.approx(exp["perplexity"], rel=1e-12)
    assert float(np.mean(effs)) == pytest.approx(exp["effective_bits"], rel=1e-15)
    assert ops == exp["estimator_ops"]
    ids = [M.LayerId.from_name(n) for n in golden_traces[f"{name}_layers"]]
    bits, est = trace_arrays(first.records, ids)
    assert np.array_equal(bits, golden_traces[f"{name}_bits"])
    np.testing.assert_allclose(est, golden_traces[f"{name}_est"], rtol=1e-12, equal_nan=True)


def test_decode_trace(report_setup, golden_traces, golden_summary):
    S = report_setup
    plan = R.load_plan(plan_path("dp_t3.5"), S.store)
    eng = oracle_engine(S.weights, S.store, plan)
    logits = eng.prefill(golden_traces["decode_prompt"])
    lg, toks = [logits], []
    for _ in range(len(golden_traces["decode_tokens"])):
        nxt = int(np.argmax(logits))
        toks.append(nxt)
        logits = eng.step(nxt)
        lg.append(logits)
    assert toks == golden_traces["decode_tokens"].tolist()
    np.testing.assert_allclose(np.array(lg), golden_traces["decode_logits"], rtol=1e-11, atol=1e-13)
    ids = [M.LayerId.from_name(n) for n in golden_traces["decode_layers"]]
    bits, _ = trace_arrays(eng.records, ids)
    assert np.array_equal(bits, golden_traces["decode_bits"])
    assert eng.estimator_ops == golden_summary["decode_estimator_ops"]


@pytest.mark.parametrize("rule", ["prev_step", "prev_block"])
def test_exact_async_plan(report_setup, golden_traces, golden_summary, rule):
    S = report_setup
    plan = R.load_plan(plan_path("exact_async_t4"), S.store)
    ppl, _, eng = oracle_eval(S.weights, S.store, plan, S.chunks[0], track_exact=True,
                              async_rule=rule)
    assert ppl == pytest.approx(golden_summary[f"exact_{rule}_perplexity"], rel=1e-12)
    ids = [M.LayerId.from_name(n) for n in golden_traces[f"exact_{rule}_layers"]]
    bits, est = trace_arrays(eng.records, ids)
    assert np.array_equal(bits, golden_traces[f"exact_{rule}_bits"])
    np.testing.assert_allclose(est, golden_traces[f"exact_{rule}_est"], rtol=1e-10, equal_nan=True)
    xids = [O.key(M.LayerId.from_name(n)) for n in golden_traces[f"exact_{rule}_xlayers"]]
    xerr = np.array([[r.exact_errors[k] for k in xids] for r in eng.records])
    np.testing.assert_allclose(xerr, golden_traces[f"exact_{rule}_xerr"], rtol=1e-10)
    assert eng.estimator_ops == golden_summary[f"exact_{rule}_estimator_ops"]


def test_linear_plan(report_setup, golden_traces, golden_summary):
    S = report_setup
    plan = R.load_plan(plan_path("linear_t3.5"), S.store)
    ppl, _, eng = oracle_eval(S.weights, S.store, plan, S.chunks[golden_summary["linear_chunk"]])
    assert ppl == pytest.approx(golden_summary["linear_perplexity"], rel=1e-12)
    ids = [M.LayerId.from_name(n) for n in golden_traces["linear_layers"]]
    bits, est = trace_arrays(eng.records, ids)
    assert np.array_equal(bits, golden_traces["linear_bits"])
    np.testing.assert_allclose(est, golden_traces["linear_est"], rtol=1e-12, equal_nan=True)
    assert eng.estimator_ops == golden_summary["linear_estimator_ops"]


def test_oracle_kv_decode_matches_batch_forward(toy_weights, toy_store):
    # reference tests/test_runtime.py:22-33 restated on the oracle
    bits = {lid: (4 if lid.kind in ("q", "k", "v") else 5) for lid in toy_store.layers}
    plan = R.sentinel_static_plan(bits, toy_store.param_counts(), 4.5)
    toks = np.random.default_rng(0).integers(0, 256, 30)
    layers = {O.key(l): O.as_layer(q) for l, q in toy_store.layers.items()}
    mats = {k: O.dequantize(layers[k], bits[M.LayerId(*k)]) for k in layers}
    logits = O.forward(toy_weights.config, toy_weights.embed, toy_weights.lm_head, lambda k: mats[k], toks)
    ppl_ref = float(np.exp(O.token_losses(logits, toks).mean()))
    ppl, _, _ = oracle_eval(toy_weights, toy_store, plan, toks)
    assert ppl == pytest.approx(ppl_ref, rel=1e-12)


def test_product_store_hash_matches_reference(tmp_path, report_setup, golden_summary):
    from paper_2508_06041_b200 import quant as Q
    p = str(tmp_path / "m.dpqs")
    Q.save_store(report_setup.store, p)
    assert Q.file_hash(p) == golden_summary["store_hash"]
    assert report_setup.weights.checksum() == golden_summary["weights_checksum"]
    back = Q.load_store(p)
    p2 = str(tmp_path / "m2.dpqs")
    Q.save_store(back, p2)
    assert Q.file_hash(p2) == golden_summary["store_hash"]
