"""Drop-in API behaviour of the device runtime (advisor findings, round 1):
plans stay plain data after an engine is built, plan edits reach the device
selector, forced bits and projection shapes are validated before any device
work, and the public API's G defaults to f32 (the reference's G is float64)."""

import copy
import os
import pickle

import numpy as np
import pytest

from paper_2508_06041_b200 import estimator as E
from paper_2508_06041_b200 import model as M
from paper_2508_06041_b200 import quant as Q
from paper_2508_06041_b200 import runtime as R

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def small():
    cfg = M.ModelConfig(n_blocks=2, d_model=64, n_heads=4, d_ff=128, seq_cap=32)
    w = M.init_model(0, cfg)
    store = Q.quantize_model(w, 6, 3)
    rng = np.random.default_rng(0)
    layers = {}
    for lid in store.ordered_ids():
        cols = store.layers[lid].shape[1]
        G = rng.standard_normal((8, cols)) * 0.1
        est = E.ErrorEstimator(E.ProjectionEstimator(G, 8, 0), E.IMMEDIATE, (3, 4))
        layers[lid] = R.PlanLayer(lid, 5, 3.5, (3, 4), 0.05, 0.5, est)
    plan = R.PrecisionPlan("dp", 3.5, 5.0, layers, store.param_counts())
    return w, store, plan


def _bits(eng, toks):
    eng.step(int(toks[0]), dynamic=False)
    for t in toks[1:]:
        eng.step(int(t))
    return np.array([[s.bits[l] for l in eng._ids] for s in eng.trace.steps])


def test_plan_stays_plain_data(small):
    w, store, plan = small
    eng = R.DecodeEngine(w, store, plan)
    eng.step(1, dynamic=False)
    assert "_device_plans" not in plan.__dict__
    copy.deepcopy(plan)
    pickle.dumps(plan)
    eng.close()


def test_plan_edits_reach_the_device(small):
    w, store, plan = small
    plan = copy.deepcopy(plan)
    toks = [3, 7, 11, 5]
    e1 = R.DecodeEngine(w, store, plan)
    assert np.all(_bits(e1, toks) == 4)          # T = 0.05: every estimate above -> high
    for pl in plan.layers.values():
        pl.T = 1e30                               # now every decision is low
    e2 = R.DecodeEngine(w, store, plan)
    assert e2.dplan is not e1.dplan
    assert np.all(_bits(e2, toks) == 3)
    e3 = R.DecodeEngine(w, store, plan)          # unchanged plan: cached selector state
    assert e3.dplan is e2.dplan
    for e in (e1, e2, e3):
        e.close()


def test_forced_bits_validated(small):
    w, store, plan = small
    eng = R.DecodeEngine(w, store, plan)
    ids = store.ordered_ids()
    eng.step(1, dynamic=False)
    with pytest.raises(ValueError):
        eng.step(2, forced_bits={ids[0]: 3})                         # layers missing
    with pytest.raises(ValueError):
        eng.step(2, forced_bits=np.full(len(ids), 7, np.int8))       # above n_bits = 6
    with pytest.raises(ValueError):
        eng.step(2, forced_bits=np.full(len(ids), -1, np.int8))
    with pytest.raises(ValueError):
        eng.step(2, forced_bits=np.full(len(ids) - 1, 4, np.int8))   # wrong length
    eng.step(2, forced_bits={l: 5 for l in ids})                    # in range: fine
    assert all(b == 5 for b in eng.trace.steps[-1].bits.values())
    eng.close()


def test_projection_shape_checked(small):
    w, store, plan = small
    bad = copy.deepcopy(plan)
    lid = store.ordered_ids()[0]
    bad.layers[lid].estimator.kind.G = np.zeros((8, 3))
    with pytest.raises(ValueError, match="projection G"):
        R.DecodeEngine(w, store, bad)


def test_public_api_defaults_to_f32_G(small):
    import inspect
    assert inspect.signature(R.DecodeEngine).parameters["g_dtype"].default == "f32"


def test_integration_stub_runs_on_reference_shaped_objects(tmp_path):
    """The ctypes stub of INTEGRATION.md §2, executed as written against
    reference-shaped objects (BitPlaneStore.layers: LayerId -> QuantizedLayer
    with codes / n_bits / b_min / lo / hi), gives the oracle's gemv."""
    import re
    import sys
    import types
    import ctypes as C
    import torch
    from oracle import dpq_oracle as O
    from paper_2508_06041_b200 import _lib
    text = open(os.path.join(os.path.dirname(__file__), "..", "INTEGRATION.md")).read()
    code = re.search(r"```python\n(# dpq/_b200\.py.*?)```", text, re.S).group(1)
    code = code.replace('C.CDLL("libdpq_b200.so")', f'C.CDLL({_lib.LIB_PATH!r})')
    fake = types.ModuleType("dpq")
    fake.model = types.ModuleType("dpq.model")
    fake.model.KINDS = M.KINDS
    sys.modules.setdefault("dpq", fake)
    sys.modules.setdefault("dpq.model", fake.model)
    ns = {}
    exec(compile(code, "INTEGRATION.md", "exec"), ns)
    cfg = M.ModelConfig(n_blocks=2, d_model=64, n_heads=4, d_ff=96, seq_cap=16)
    store = Q.quantize_model(M.init_model(1, cfg), 5, 3)
    handle, index = ns["device_store"](store)
    rng = np.random.default_rng(2)
    for lid in list(store.layers)[::3]:
        q = store.layers[lid]
        x = torch.as_tensor(rng.standard_normal(q.shape[1]), dtype=torch.float32, device="cuda")
        y = torch.empty(q.shape[0], dtype=torch.float32, device="cuda")
        ns["gemv"](handle, index, lid, 4, x.data_ptr(), y.data_ptr())
        torch.cuda.synchronize()
        ref = O.gemv(O.as_layer(q), 4, x.double().cpu().numpy())
        np.testing.assert_allclose(y.cpu().numpy(), ref, rtol=0, atol=1e-5 * np.abs(ref).max())
    _lib.load().dpq_store_destroy(handle)


def test_fixed_point_range_is_flagged(small):
    """Activations far outside the fixed-point range of the engine's packed
    partial sums / estimator words (|S_w| >= 2^33, |G.x| 2^fb >= 2^47) raise
    DeviceError (DPQ_ERR_RANGE) instead of wrapping silently."""
    from paper_2508_06041_b200 import _lib
    w, store, plan = small
    big = M.ModelWeights(w.config, w.embed * np.float32(1e9), w.lm_head, w.linears)
    eng = R.DecodeEngine(big, store, plan)
    assert _lib.load().dpq_session_is_persistent(eng._h) == 2
    with pytest.raises(_lib.DeviceError, match="range"):
        eng.step(1, dynamic=False)
        eng.step(2, dynamic=True)
    eng.close()
