"""Device store / GEMV / selector parity against the oracle (GPU).

Tolerances: dequantize bit-exact (same float64 IEEE
ops); GEMV max|y - y_ref| <= 1e-5 * max|y_ref| (float32 LUT path vs float64
reference); estimates rel 1e-5 (f32 G) / 2e-3 (f16 G); decisions bit-exact
except within eps*|T| of the threshold.
"""

import numpy as np
import pytest
import torch

from oracle import dpq_oracle as O
from paper_2508_06041_b200 import _lib
from paper_2508_06041_b200 import estimator as E
from paper_2508_06041_b200 import quant as Q
from paper_2508_06041_b200 import runtime as R
from paper_2508_06041_b200.model import LayerId

pytestmark = pytest.mark.gpu
GEMV_TOL = 1e-5


def close_y(y, y_ref, tol=GEMV_TOL):
    err = np.max(np.abs(np.asarray(y, dtype=np.float64) - y_ref))
    assert err <= tol * max(np.max(np.abs(y_ref)), 1e-30), (err, np.max(np.abs(y_ref)))


def golden_layer(g, case):
    r, c, n, bmin = (int(v) for v in g[f"c{case}_meta"])
    return Q.QuantizedLayer(g[f"c{case}_codes"].astype(np.uint16), n, bmin, g[f"c{case}_lo"],
                            g[f"c{case}_hi"]), r, c, n, bmin


@pytest.mark.parametrize("case", range(6))
def test_dequantize_bit_exact_and_gemv(quant_vectors, case):
    q, r, c, n, bmin = golden_layer(quant_vectors, case)
    x = quant_vectors[f"c{case}_x"]
    for b in range(bmin, n + 1):
        d = Q.dequantize(q, b)
        assert np.array_equal(d, O.dequantize(O.as_layer(q), b))
        if quant_vectors[f"c{case}_deq{b}"].size:
            assert np.array_equal(d, quant_vectors[f"c{case}_deq{b}"])
        close_y(Q.gemv(q, b, x), quant_vectors[f"c{case}_y{b}"])


def test_kat_two_bit_device():
    q = Q.quantize_layer(np.array([[0.0, 0.3, 0.6, 1.0]]), 2, 2)
    np.testing.assert_array_equal(Q.dequantize(q, 2), [[0.125, 0.375, 0.625, 0.875]])
    close_y(Q.gemv(q, 2, np.array([1.0, 2.0, 3.0, 4.0])), np.array([0.125 + 0.75 + 1.875 + 3.5]))


def test_degenerate_row_reconstructs_exactly():
    q = Q.quantize_layer(np.array([[2.5, 2.5, 2.5], [0.0, 1.0, 2.0]]), 4, 3)
    for b in (3, 4):
        assert np.all(Q.dequantize(q, b)[0] == 2.5)
        y = Q.gemv(q, b, np.array([1.0, -2.0, 0.5]))
        assert abs(y[0] - 2.5 * (-0.5)) <= 1e-6


@pytest.mark.parametrize("shape", [(4096, 4096), (14336, 4096), (4096, 14336)])
def test_cfg2_gemv_all_bits(shape):
    """W ~ N(0, 1/cols), 8-bit store, b = 3..8."""
    rows, cols = shape
    rng = np.random.default_rng(rows + cols)
    W = rng.normal(0.0, 1.0 / np.sqrt(cols), shape).astype(np.float32)
    q = Q.quantize_layer(W, 8, 3)
    x = rng.normal(size=cols)
    x = x / np.sqrt(np.mean(x * x) + 1e-6)
    ol = O.as_layer(q)
    xt = torch.as_tensor(x.astype(np.float32), device="cuda")
    for b in range(3, 9):
        y = Q.gemv(q, b, xt).double().cpu().numpy()
        close_y(y, O.plane_sum_gemv(ol, b, x.astype(np.float32).astype(np.float64)))


def test_quantize_device_bit_identical():
    rng = np.random.default_rng(5)
    W = rng.normal(0, 0.05, (300, 700)).astype(np.float32)
    W[7] = 0.125
    for n in (4, 6, 8):
        ref = Q.quantize_layer(W, n, 3)
        Wd = torch.as_tensor(W, device="cuda")
        codes = torch.empty((300, 700), dtype=torch.int16, device="cuda")
        lo = torch.empty(300, device="cuda")
        hi = torch.empty(300, device="cuda")
        _lib.call("dpq_quantize_device", 0, Wd.data_ptr(), 300, 700, n, codes.data_ptr(),
                  lo.data_ptr(), hi.data_ptr(), None)
        torch.cuda.synchronize()
        assert np.array_equal(codes.cpu().numpy().view(np.uint16), ref.codes)
        assert np.array_equal(lo.cpu().numpy(), ref.lo) and np.array_equal(hi.cpu().numpy(), ref.hi)


def test_exact_error_device(quant_vectors):
    for case in (0, 1, 2, 5):
        q, r, c, n, bmin = golden_layer(quant_vectors, case)
        x = quant_vectors[f"c{case}_x"]
        got = E.exact_error(q, bmin, bmin + 1, x)
        assert got == pytest.approx(quant_vectors[f"c{case}_exact"][0], rel=1e-5)
        assert E.exact_error(q, bmin, n, x) == pytest.approx(O.exact_error(O.as_layer(q), bmin, n, x), rel=1e-5)


def _select(q, pl, x, g_dtype="f32", est_in=None, want_exact=False):
    ds = Q.DeviceStore([q])
    dp = R.DevicePlan(ds, [pl], g_dtype)
    xt = torch.as_tensor(np.asarray(x, dtype=np.float32), device="cuda")
    ei = torch.as_tensor(np.asarray(est_in, dtype=np.float32), device="cuda") if est_in is not None else None
    y = torch.empty(q.shape[0], device="cuda")
    bit = torch.zeros(1, dtype=torch.int32, device="cuda")
    est = torch.zeros(1, device="cuda")
    ex = torch.zeros(1, device="cuda")
    _lib.call("dpq_select_gemv", dp.handle, 0, xt.data_ptr(), ei.data_ptr() if ei is not None else None,
              y.data_ptr(), bit.data_ptr(), est.data_ptr(), ex.data_ptr() if want_exact else None,
              _lib.stream_ptr())
    torch.cuda.synchronize()
    return y.double().cpu().numpy(), int(bit.item()), float(est.item()), float(ex.item())


def _proj_layer(rows=200, cols=700, seed=3, k=64):
    rng = np.random.default_rng(seed)
    q = Q.quantize_layer(rng.normal(0, 1 / np.sqrt(cols), (rows, cols)), 6, 3)
    A = rng.standard_normal((k, rows)) / np.sqrt(k)
    G = A @ O.delta_weights(O.as_layer(q), 3, 4)
    return q, G, rng


@pytest.mark.parametrize("g_dtype,tol", [("f32", 1e-5), ("f16", 2e-3), ("e4m3", 5e-2)])
def test_select_gemv_projection(g_dtype, tol):
    q, G, rng = _proj_layer()
    lid = LayerId(0, "q")
    est_obj = E.ErrorEstimator(E.ProjectionEstimator(G, 64, 0), E.IMMEDIATE, (3, 4))
    x = rng.normal(size=700)
    ref_est = float(np.linalg.norm(G @ x.astype(np.float32).astype(np.float64)))
    ol = O.as_layer(q)
    for T, want in ((ref_est * 0.9, 4), (ref_est * 1.1, 3)):
        pl = R.PlanLayer(lid, 6, 3.5, (3, 4), T, 0.5, est_obj)
        y, bit, est, _ = _select(q, pl, x, g_dtype)
        assert bit == want
        assert est == pytest.approx(ref_est, rel=tol)
        close_y(y, O.gemv(ol, bit, x.astype(np.float32)))
    # the standalone estimator API agrees
    assert est_obj.estimate(x) == pytest.approx(ref_est, rel=1e-6)


def test_select_gemv_linear_and_sentinels():
    q, G, rng = _proj_layer(seed=4)
    lid = LayerId(0, "up")
    x = rng.normal(size=700)
    nx = float(np.linalg.norm(x.astype(np.float32)))
    lin = E.ErrorEstimator(E.LinearEstimator(0.3, 0.1, 0.95), E.IMMEDIATE, (3, 5))
    ref = 0.3 * nx + 0.1
    for T, want in ((ref - 1e-3, 5), (ref + 1e-3, 3)):
        y, bit, est, _ = _select(q, R.PlanLayer(lid, 6, 4.0, (3, 5), T, 0.5, lin), x)
        assert bit == want and est == pytest.approx(ref, rel=1e-6)
        close_y(y, O.gemv(O.as_layer(q), want, x.astype(np.float32)))
    y, bit, est, _ = _select(q, R.PlanLayer(lid, 6, 4.0, (3, 5), np.inf, 1.0, None), x)
    assert bit == 3 and np.isnan(est)
    y, bit, est, _ = _select(q, R.PlanLayer(lid, 6, 4.0, (3, 5), -np.inf, 0.0, None), x)
    assert bit == 5 and np.isnan(est)


def test_select_gemv_async_input_and_exact():
    q, G, rng = _proj_layer(seed=5)
    lid = LayerId(1, "q")
    x, xp = rng.normal(size=700), rng.normal(size=700)
    ol = O.as_layer(q)
    xp32 = xp.astype(np.float32).astype(np.float64)
    x32 = x.astype(np.float32).astype(np.float64)
    # projection on the previous input
    proj = E.ErrorEstimator(E.ProjectionEstimator(G, 64, 0), E.PREVIOUS_RESIDUAL, (3, 4))
    ref = float(np.linalg.norm(G @ xp32))
    y, bit, est, ex = _select(q, R.PlanLayer(lid, 6, 3.5, (3, 4), ref * 0.95, 0.5, proj), x, est_in=xp,
                              want_exact=True)
    assert bit == 4 and est == pytest.approx(ref, rel=1e-5)
    assert ex == pytest.approx(O.exact_error(ol, 3, 4, x32), rel=1e-5)
    close_y(y, O.gemv(ol, 4, x32))
    # exact estimator, immediate and on the previous input
    exact = E.ErrorEstimator(E.ExactEstimator(q, 3, 4), E.IMMEDIATE, (3, 4))
    e_now = O.exact_error(ol, 3, 4, x32)
    y, bit, est, _ = _select(q, R.PlanLayer(lid, 6, 3.5, (3, 4), e_now * 1.01, 0.5, exact), x)
    assert bit == 3 and est == pytest.approx(e_now, rel=1e-5)
    close_y(y, O.gemv(ol, 3, x32))
    e_prev = O.exact_error(ol, 3, 4, xp32)
    y, bit, est, _ = _select(q, R.PlanLayer(lid, 6, 3.5, (3, 4), e_prev * 0.99, 0.5, exact), x, est_in=xp)
    assert bit == 4 and est == pytest.approx(e_prev, rel=1e-5)
    close_y(y, O.gemv(ol, 4, x32))


def test_select_precision_api_matches_oracle(toy_store):
    lid = LayerId(0, "q")
    layer = toy_store.layers[lid]
    est = E.ErrorEstimator(E.ExactEstimator(layer, 3, 4), E.IMMEDIATE, (3, 4))
    x = np.random.default_rng(1).normal(size=32)
    err = O.exact_error(O.as_layer(layer), 3, 4, x)
    assert R.select_precision(R.PlanLayer(lid, 6, 3.5, (3, 4), err * 2, 0.5, est), x)[0] == 3
    bit, e, cost = R.select_precision(R.PlanLayer(lid, 6, 3.5, (3, 4), err / 2, 0.5, est), x)
    assert bit == 4 and e == pytest.approx(err, rel=1e-5) and cost == 32 * 32


@pytest.mark.parametrize("shape,pair", [((200, 700), (3, 4)), ((1000, 96), (4, 6))])
def test_build_projection_on_device_matches_oracle(shape, pair):
    """estimator.py:190-200 with dW dequantized on the device (fp64) and the
    A @ dW product formed by the GPU: equals the oracle's host product."""
    rng = np.random.default_rng(shape[0])
    q = Q.quantize_layer(rng.normal(0, 1 / np.sqrt(shape[1]), shape), 6, 3)
    l, h = pair
    est = E.build_projection(q, l, h, 64, seed=9)
    assert isinstance(est, E.ProjectionEstimator) and (est.k, est.seed) == (64, 9)
    G = est.G
    G_ref = O.build_projection_G(O.as_layer(q), l, h, 64, 9)
    assert G.shape == (64, shape[1])
    np.testing.assert_allclose(G, G_ref, rtol=1e-10, atol=1e-12 * np.abs(G_ref).max())


@pytest.mark.parametrize("shape", [(45, 700), (100, 512), (1000, 96), (4128, 1500), (96, 40 * 512 + 7),
                                   (33, 9000)])
def test_gemv_kernel_ragged_shapes(shape, monkeypatch):
    """bitplane_gemv_kernel (csrc/dpq_gemv.cu) on ragged shapes: fewer tasks
    than CTAs, rows not a multiple of 32, partial windows, CTA ranges over two
    windows (few tiles per window): equal to the oracle at every b, and to the
    single-op engine program (DPQ_GEMV_KERNEL=0); repeated calls (the
    self-resetting tile counters) give identical results."""
    rows, cols = shape
    rng = np.random.default_rng(rows * 7 + cols)
    W = rng.normal(0.0, 1.0 / np.sqrt(cols), shape)
    q = Q.quantize_layer(W, 6, 3)
    x = rng.normal(size=cols).astype(np.float32)
    ol = O.as_layer(q)
    xt = torch.as_tensor(x, device="cuda")
    for b in range(3, 7):
        y1 = Q.gemv(q, b, xt).double().cpu().numpy()
        y2 = Q.gemv(q, b, xt).double().cpu().numpy()
        assert np.array_equal(y1, y2)
        close_y(y1, O.plane_sum_gemv(ol, b, x.astype(np.float64)))
    monkeypatch.setenv("DPQ_GEMV_KERNEL", "0")
    y3 = Q.gemv(q, 5, xt).double().cpu().numpy()
    monkeypatch.delenv("DPQ_GEMV_KERNEL")
    close_y(Q.gemv(q, 5, xt).double().cpu().numpy(), y3)


@pytest.mark.parametrize("cols", [700, 4100])
def test_gemv_kernel_selector_matches_engine_program(cols, monkeypatch):
    """dpq_select_gemv through bitplane_gemv_kernel (projection selector, f32
    G, pair (3, 5)) and through the single-op engine program: same bit, same
    estimate (the same fixed-point G.x sums), outputs within the GEMV tolerance."""
    rng = np.random.default_rng(cols)
    rows = 300
    W = rng.normal(0.0, 1.0 / np.sqrt(cols), (rows, cols))
    q = Q.quantize_layer(W, 6, 3)
    G = rng.normal(size=(64, cols)) / np.sqrt(cols)
    x = rng.normal(size=cols)
    ref_est = float(np.linalg.norm(G @ x.astype(np.float32).astype(np.float64)))
    est_obj = E.ErrorEstimator(E.ProjectionEstimator(G, 64, 0), E.IMMEDIATE, (3, 5))
    for T, want in ((ref_est * 0.99, 5), (ref_est * 1.01, 3)):
        pl = R.PlanLayer(LayerId(0, "o"), 6, 4.0, (3, 5), T, 0.5, est_obj)
        outs = []
        for env in ("1", "0"):
            monkeypatch.setenv("DPQ_GEMV_KERNEL", env)
            outs.append(_select(q, pl, x, "f32"))
        monkeypatch.delenv("DPQ_GEMV_KERNEL")
        (y1, b1, e1, _), (y2, b2, e2, _) = outs
        assert b1 == b2 == want
        assert e1 == e2 and e1 == pytest.approx(ref_est, rel=1e-5)
        close_y(y1, np.asarray(y2, dtype=np.float64))
        close_y(y1, O.gemv(O.as_layer(q), want, x.astype(np.float32)))


@pytest.mark.parametrize("shape", [(14336, 4096), (4096, 14336)])
def test_gemv_kernel_selector_large_layers(shape, monkeypatch):
    """dpq_select_gemv on cfg2 shapes (projection selector, f32 G, pair (3, 4)):
    more than one wave of chunk groups per CTA, so the decided bits stream
    base and extra planes together after the first wave. Bit, estimate and
    output against the oracle, both decisions."""
    rows, cols = shape
    rng = np.random.default_rng(rows + 3 * cols)
    W = rng.normal(0.0, 1.0 / np.sqrt(cols), shape)
    q = Q.quantize_layer(W, 4, 3)
    G = rng.normal(size=(64, cols)) / np.sqrt(cols)
    x = rng.normal(size=cols)
    ref_est = float(np.linalg.norm(G @ x.astype(np.float32).astype(np.float64)))
    est_obj = E.ErrorEstimator(E.ProjectionEstimator(G, 64, 0), E.IMMEDIATE, (3, 4))
    ol = O.as_layer(q)
    for T, want in ((ref_est * 0.99, 4), (ref_est * 1.01, 3)):
        pl = R.PlanLayer(LayerId(0, "up"), 4, 3.5, (3, 4), T, 0.5, est_obj)
        y, bit, est, _ = _select(q, pl, x, "f32")
        assert bit == want
        assert est == pytest.approx(ref_est, rel=1e-5)
        close_y(y, O.plane_sum_gemv(ol, want, x.astype(np.float32).astype(np.float64)))
