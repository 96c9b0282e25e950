"""model.forward / teacher_forced_loss / backward drop-ins (reference
model.py:286-460, re-exported by dpq/__init__.py:8-10) as fp64 device
graphs, against vectors the reference produced (tools/make_golden.py
model_vectors): full-precision and 4-bit dequantized providers."""

import os

import numpy as np
import pytest

import paper_2508_06041_b200 as D
from paper_2508_06041_b200 import model as M
from paper_2508_06041_b200 import quant as Q

from conftest import GOLDEN

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["fp", "q4"])
def test_forward_backward_match_reference(name):
    g = dict(np.load(os.path.join(GOLDEN, "model_vectors.npz")))
    mc = M.ModelConfig(n_blocks=2, d_model=32, n_heads=4, d_ff=64, vocab=256, seq_cap=64)
    w = M.init_model(0, mc)
    store = Q.quantize_model(w, 6, 3)
    prov = None if name == "fp" else (lambda lid: Q.dequantize(store.layers[lid], 4))
    toks = g["tokens"]
    lg, tape = D.forward(w, toks, prov, want_tape=True)
    np.testing.assert_allclose(lg, g[f"{name}/logits"], rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(tape.x_final, g[f"{name}/x_final"], rtol=1e-10, atol=1e-12)
    for b, bt in enumerate(tape.blocks):
        for f in ("n1", "attn_cat", "h", "probs", "x_mid"):
            np.testing.assert_allclose(getattr(bt, f), g[f"{name}/b{b}/{f}"], rtol=1e-9, atol=1e-12)
    loss, ppl, per = D.teacher_forced_loss(w, toks, prov)
    np.testing.assert_allclose([loss, ppl], g[f"{name}/tfl"], rtol=1e-11)
    np.testing.assert_allclose(per, g[f"{name}/per_token"], rtol=1e-10)
    bl, bundle, _ = D.backward(w, toks, prov)
    np.testing.assert_allclose(bl, g[f"{name}/bwd_loss"][0], rtol=1e-11)
    for lid in M.layer_ids(mc):
        ref_w, ref_o = g[f"{name}/wg/{lid.name}"], g[f"{name}/og/{lid.name}"]
        np.testing.assert_allclose(bundle.weight_grads[lid], ref_w, rtol=1e-7, atol=1e-10 * np.abs(ref_w).max())
        np.testing.assert_allclose(bundle.output_grads[lid], ref_o, rtol=1e-7, atol=1e-10 * np.abs(ref_o).max())
    with pytest.raises(ValueError):
        D.backward(w, toks[:1])
