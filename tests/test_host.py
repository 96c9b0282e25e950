"""Host-side logic and the C-ABI surface (CPU only, no device calls)."""

import ctypes as C
import os
import re

import numpy as np
import pytest

from oracle import dpq_oracle as O
from paper_2508_06041_b200 import _lib
from paper_2508_06041_b200 import model as M
from paper_2508_06041_b200 import quant as Q
from paper_2508_06041_b200 import runtime as R
from conftest import ROOT, TOY, plan_path


def header_functions():
    src = open(os.path.join(ROOT, "include", "dpq_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|const char\*)\s+(dpq_\w+)\(", src, re.M)))


def test_library_exports_every_header_symbol():
    lib = _lib.load()
    names = header_functions()
    assert len(names) >= 25
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(_lib.EXPORTED)
    assert lib.dpq_version() == 1


def numpy_repack(codes, n_bits):
    """Independent restatement of the device plane layout (dpq_common.cuh)."""
    rows, cols = codes.shape
    nt, nw = -(-rows // 32), -(-cols // 512)
    c = np.zeros((nt * 32, nw * 512), dtype=np.uint16)
    c[:rows, :cols] = codes
    out = np.zeros((n_bits, nw, nt, 4, 32, 16), dtype=np.uint8)
    lane = np.arange(32)
    for p in range(n_bits):
        bit = ((c >> (n_bits - 1 - p)) & 1).astype(np.uint16)
        # byte of group g: bit t -> column 8g+t
        by = np.zeros((nt * 32, nw, 64), dtype=np.uint16)
        for t in range(8):
            by |= bit.reshape(nt * 32, nw, 64, 8)[..., t] << t
        for s in range(64):
            g = (lane + s) % 64
            wrap = (lane + s >= 64).astype(np.uint16)
            for tile in range(nt):
                rowsel = tile * 32 + lane
                e = (by[rowsel, :, g] - wrap[:, None]) & 255    # [lane, window]
                out[p, :, tile, s // 16, :, s % 16] = e.T
    return out.reshape(-1)


@pytest.mark.parametrize("shape,n_bits", [((37, 53), 6), ((64, 1100), 4), ((5, 512), 8), ((96, 40), 3)])
def test_repack_layout_host(shape, n_bits):
    rng = np.random.default_rng(sum(shape) + n_bits)
    codes = rng.integers(0, 1 << n_bits, size=shape).astype(np.uint16)
    nbytes = _lib.load().dpq_planes_bytes(shape[0], shape[1], n_bits)
    buf = np.zeros(nbytes, dtype=np.uint8)
    _lib.call("dpq_repack_host", codes.ctypes.data, shape[0], shape[1], n_bits,
              buf.ctypes.data, C.c_int64(nbytes))
    assert np.array_equal(buf, numpy_repack(codes, n_bits))


def lut_gemv_model(codes, lo, hi, n_bits, b, x):
    """Float64 model of the kernel's arithmetic on the packed planes: byte LUT
    lookups with the rotated-slot address trick, Horner over planes, affine
    epilogue. Proves the layout + address trick compute W_b x."""
    rows, cols = codes.shape
    nbytes = _lib.load().dpq_planes_bytes(rows, cols, n_bits)
    planes = np.zeros(nbytes, dtype=np.uint8)
    _lib.call("dpq_repack_host", codes.ctypes.data, rows, cols, n_bits, planes.ctypes.data,
              C.c_int64(nbytes))
    nt, nw = -(-rows // 32), -(-cols // 512)
    planes = planes.reshape(n_bits, nw, nt, 4, 32, 16)
    xp = np.zeros(nw * 512)
    xp[:cols] = x
    S = np.zeros(nt * 32)
    lane = np.arange(32)
    for w in range(nw):
        xg = xp[w * 512:(w + 1) * 512].reshape(64, 8)
        lut = np.zeros((257, 64))
        for e in range(256):
            bits = (e >> np.arange(8)) & 1
            lut[e] = xg @ bits
        for tile in range(nt):
            Sw = np.zeros(32)
            for p in range(b):
                P = np.zeros(32)
                for s in range(64):
                    byte = planes[p, w, tile, s // 16, :, s % 16].astype(np.int64)
                    addr = (byte << 8) + 4 * lane + 4 * s        # byte address in the LUT
                    P += lut.reshape(-1)[addr // 4]
                Sw = 2 * Sw + P
            S[tile * 32:(tile + 1) * 32] += Sw
    S = S[:rows]
    sx = x.sum()
    span = hi.astype(np.float64) - lo.astype(np.float64)
    return lo.astype(np.float64) * sx + span / (1 << b) * (S + 0.5 * sx)


@pytest.mark.parametrize("case", [0, 2, 3])
def test_lut_address_trick_matches_oracle(quant_vectors, case):
    g = quant_vectors
    r, c, n, bmin = (int(v) for v in g[f"c{case}_meta"])
    codes = g[f"c{case}_codes"].astype(np.uint16)
    for b in (bmin, n):
        y = lut_gemv_model(codes, g[f"c{case}_lo"], g[f"c{case}_hi"], n, b, g[f"c{case}_x"])
        np.testing.assert_allclose(y, g[f"c{case}_y{b}"], rtol=1e-9, atol=1e-9)


def test_quantize_layer_bit_identical_to_oracle(quant_vectors):
    for case in range(6):
        if f"c{case}_W" not in quant_vectors:
            continue
        r, c, n, bmin = (int(v) for v in quant_vectors[f"c{case}_meta"])
        q = Q.quantize_layer(quant_vectors[f"c{case}_W"], n, bmin)
        assert np.array_equal(q.codes, quant_vectors[f"c{case}_codes"])
        assert np.array_equal(q.lo, quant_vectors[f"c{case}_lo"])


def test_quant_errors_raised_before_device():
    q = Q.quantize_layer(np.ones((2, 3)), 6, 3)
    with pytest.raises(Q.QuantError):
        Q.dequantize(q, 2)
    with pytest.raises(Q.QuantError):
        Q.dequantize(q, 7)
    with pytest.raises(Q.QuantError):
        Q.gemv(q, 4, np.zeros(5))
    with pytest.raises(Q.QuantError):
        Q.delta_weights(q, 5, 5)
    with pytest.raises(Q.QuantError):
        Q.quantize_layer(np.ones((2, 2)), 9, 3)
    with pytest.raises(Q.QuantError):
        Q.quantize_layer(np.array([[np.nan, 1.0]]), 6, 3)


def test_pack_round_trip_matches_oracle():
    rng = np.random.default_rng(4)
    for n_bits in (3, 5, 6, 8):
        codes = rng.integers(0, 1 << n_bits, size=(7, 13)).astype(np.uint16)
        blob = Q.pack_codes(codes, n_bits)
        assert blob == O.pack_codes(codes, n_bits)
        assert np.array_equal(Q.unpack_codes(blob, n_bits, codes.shape), codes)


def test_store_rejects_wrong_magic(tmp_path):
    p = str(tmp_path / "bad.dpqs")
    open(p, "wb").write(b"NOPE" + b"\x00" * 64)
    with pytest.raises(Q.QuantError):
        Q.load_store(p)


def test_config_hash_and_gqa_extension():
    import sys
    assert TOY.hash() == M.ModelConfig(2, 32, 4, 64, seq_cap=64, n_kv_heads=4).hash()
    g = M.ModelConfig(2, 64, 8, 96, n_kv_heads=2)
    assert M.layer_shape(g, M.LayerId(0, "k")) == (16, 64)
    assert "n_kv_heads" in g.to_dict()
    with pytest.raises(ValueError):
        M.ModelConfig(2, 64, 8, 96, n_kv_heads=3)


def test_layer_id_interop():
    a = M.LayerId(1, "q")
    assert a == M.LayerId.from_name("block1.q")
    assert {a: 1}[M.LayerId(1, "q")] == 1
    with pytest.raises(ValueError):
        M.LayerId(0, "nope")


def test_plan_round_trip_and_reference_files(tmp_path, report_setup):
    for name in ("dp_t3.5", "llm_mq_t3.5", "exact_async_t4", "linear_t3.5"):
        plan = R.load_plan(plan_path(name), report_setup.store)
        p = str(tmp_path / f"{name}.json")
        R.save_plan(plan, p)
        back = R.load_plan(p, report_setup.store)
        for lid, pl in plan.layers.items():
            bl = back.layers[lid]
            assert bl.pair == pl.pair and bl.prefill_bit == pl.prefill_bit
            assert bl.T == pl.T
    with pytest.raises(ValueError):
        R.load_plan(plan_path("exact_async_t4"))      # exact plan needs the store


def test_engine_validation_before_device(toy_weights, toy_store):
    plan = R.sentinel_static_plan({l: 4 for l in toy_store.layers}, toy_store.param_counts(), 4.0)
    plan.store_hash = "deadbeef" * 8
    with pytest.raises(R.ProvenanceError):
        R.DecodeEngine(toy_weights, toy_store, plan, store_hash="feed" * 16)
    other = M.init_model(0, M.ModelConfig(n_blocks=1, d_model=32, n_heads=4, d_ff=64, seq_cap=64))
    with pytest.raises(R.ProvenanceError):
        R.DecodeEngine(other, toy_store, plan)
    plan.store_hash = ""
    with pytest.raises(ValueError):
        R.DecodeEngine(toy_weights, toy_store, plan, async_rule="nope")
    with pytest.raises(ValueError):
        R.decode(toy_weights, toy_store, plan, [], 3)
    for args in (([1], "fp"), ([1, 2], "nope"), ([1, 2], "dynamic"), ([1, 2], "static")):
        with pytest.raises(ValueError):
            R.eval_perplexity(toy_weights, toy_store, args[0], args[1])


def test_select_precision_sentinels_host():
    lid = M.LayerId(0, "q")
    assert R.select_precision(R.PlanLayer(lid, 6, 3.5, (3, 4), np.inf, 1.0, None), np.zeros(32)) == (3, None, 0)
    assert R.select_precision(R.PlanLayer(lid, 6, 3.5, (3, 4), -np.inf, 0.0, None), np.zeros(32)) == (4, None, 0)


def test_qos_and_trace_helpers(tmp_path):
    traces = []
    for eff in [3.0, 3.5, 4.0, 4.5, 5.0]:
        t = R.DecodeTrace()
        t.steps.append(R.StepRecord(0, {M.LayerId(0, "q"): 3}, {M.LayerId(0, "q"): None}, {}, eff))
        traces.append(t)
    qs = R.qos_stats(traces, 4.0)
    assert np.isclose(qs["mean"], 4.0) and qs["p90"] == 5.0 and np.isclose(qs["p90_delta_pct"], 25.0)
    assert qs == O.qos_stats([3.0, 3.5, 4.0, 4.5, 5.0], 4.0)
    with pytest.raises(ValueError):
        R.qos_stats([], 4.0)
    p = str(tmp_path / "t.csv")
    traces[0].export_csv(p)
    assert open(p).read().splitlines() == ["step,layer,bit,estimate", "0,block0.q,3,"]


def test_translate_threshold_matches_oracle():
    """estimator.py:94-121 (threshold translation for offline calibration):
    lattice quantiles, the +/-inf sentinels at r = 1 / r = 0, argument errors."""
    from paper_2508_06041_b200 import estimator as E
    rng = np.random.default_rng(4)
    for n in (1, 7, 10, 64, 257):
        errs = np.sort(rng.random(n))
        for l in (3, 4):
            for frac in (0.0, 0.1, 0.3, 0.5, 1 / 3, 0.7, 0.99, 1.0):
                p = l + frac
                e = E.translate_threshold(errs, p, l)
                assert (e.T, e.r_quantile) == O.translate_threshold(errs, p, l)
                assert e.pair == (l, l + 1) and e.layer is None
    assert E.translate_threshold([0.5], 3.0, 3).T == np.inf
    assert E.translate_threshold([0.5], 4.0, 3).T == -np.inf
    with pytest.raises(ValueError):
        E.translate_threshold([], 3.5, 3)
    with pytest.raises(ValueError):
        E.translate_threshold([0.1], 4.5, 3)


def test_threshold_oracle_pinned_to_reference():
    """The oracle's quantile / translation equal the reference's own functions
    (run here only, where /root/reference exists)."""
    import importlib
    import sys
    src = "/root/reference/pkg/src"
    if not os.path.isdir(src):
        pytest.skip("reference not present")
    sys.path.insert(0, src)
    try:
        ref = importlib.import_module("dpq.estimator")
    finally:
        sys.path.remove(src)
    rng = np.random.default_rng(5)
    for n in (1, 10, 33):
        errs = np.sort(rng.random(n))
        for frac in (0.0, 0.3, 0.5, 0.7, 1.0):
            e = ref.translate_threshold(errs, 3 + frac, 3)
            assert (e.T, e.r_quantile) == O.translate_threshold(errs, 3 + frac, 3)
