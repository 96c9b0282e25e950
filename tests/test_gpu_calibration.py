"""Offline calibration on the GPU against vectors the
unmodified reference produced (tools/make_golden.py calib_vectors):
collect_error_samples (estimator.py:132-165), calibrate_projection
(estimator.py:208-264), fit_linear (estimator.py:168-187). Same model,
store, pairs and calibration chunks; fp64 on both sides, so only summation
order differs."""

import os

import numpy as np
import pytest

from paper_2508_06041_b200 import estimator as E
from paper_2508_06041_b200 import model as M
from paper_2508_06041_b200 import quant as Q

from conftest import GOLDEN

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def calib_setup():
    g = dict(np.load(os.path.join(GOLDEN, "calib_vectors.npz")))
    mc = M.ModelConfig(n_blocks=2, d_model=64, n_heads=4, d_ff=128, vocab=256, seq_cap=64)
    w = M.init_model(3, mc)
    store = Q.quantize_model(w, 6, 3)
    ids = M.layer_ids(mc)
    pairs = {lid: ((3, 4) if i % 2 == 0 else (4, 5)) for i, lid in enumerate(ids)}
    samples = E.collect_error_samples(w, store, pairs, {lid: 5 for lid in ids}, list(g["calib"]))
    return g, store, ids, pairs, samples


def test_collect_error_samples_matches_reference(calib_setup):
    g, store, ids, pairs, samples = calib_setup
    for lid in ids:
        s = samples[lid]
        np.testing.assert_allclose(s.inputs, g[f"{lid.name}/inputs"], rtol=1e-9, atol=1e-12)
        np.testing.assert_allclose(s.errors, g[f"{lid.name}/errors"], rtol=1e-9, atol=1e-14)
        np.testing.assert_allclose(s.norms, g[f"{lid.name}/norms"], rtol=1e-12)
        np.testing.assert_array_equal(s.sorted_errors, np.sort(s.errors))


def test_calibrate_projection_matches_reference(calib_setup):
    g, store, ids, pairs, samples = calib_setup
    for lid in (ids[0], ids[6]):
        l, h = pairs[lid]
        est = E.build_projection(store.layers[lid], l, h, 8, 5)
        np.testing.assert_allclose(est.G, g[f"{lid.name}/G0"], rtol=1e-10, atol=1e-14)
        cal, hist, warn = E.calibrate_projection(est, samples[lid].inputs, samples[lid].errors, epochs=40)
        ref_hist = g[f"{lid.name}/history"]
        assert len(hist) == len(ref_hist) and int(warn) == int(g[f"{lid.name}/warning"][0])
        np.testing.assert_allclose(hist, ref_hist, rtol=1e-6)
        np.testing.assert_allclose(cal.G, g[f"{lid.name}/G"], rtol=1e-6, atol=1e-9 * np.abs(cal.G).max())
        assert cal.calibrated and hist[-1] < hist[0]
        lin = E.fit_linear(samples[lid].errors, samples[lid].norms)
        ref = g[f"{lid.name}/linear"]
        if np.isnan(ref[0]):
            assert lin is None
        else:
            np.testing.assert_allclose([lin.slope, lin.intercept, lin.r2], ref, rtol=1e-9)
