"""``.dpqs`` store file straight into device bitplanes.

``load_device_store`` uploads each layer's packed code stream (quant.py:123-126,
code-major LSB-first) and repacks it on the device. The planes must be
bit-identical to the ones built from host uint16 codes (``load_store`` ->
``dpq_store_create(code_bytes=2)``), for every n_bits (codes straddling byte
boundaries at 3/5/6/7 bits) and ragged shapes; and a decode over the
reference's own store file must equal the host-loaded one exactly.
"""

import numpy as np
import pytest
import torch

from conftest import plan_path
from paper_2508_06041_b200 import model as M
from paper_2508_06041_b200 import quant as Q
from paper_2508_06041_b200 import runtime as R

@pytest.mark.gpu
@pytest.mark.parametrize("n_bits,b_min", [(3, 2), (4, 3), (5, 3), (6, 3), (7, 4), (8, 3)])
def test_packed_upload_bit_identical(tmp_path, n_bits, b_min):
    rng = np.random.default_rng(n_bits)
    shapes = [(33, 517), (70, 1030), (1, 9), (96, 512)]          # ragged rows/cols, tiny, aligned
    layers = {}
    for b, (r, c) in enumerate(shapes):
        layers[M.LayerId(b, "q")] = Q.quantize_layer(rng.standard_normal((r, c)), n_bits, b_min)
    store = Q.BitPlaneStore(layers, n_bits, b_min, "0" * 64)
    p = str(tmp_path / "s.dpqs")
    Q.save_store(store, p)
    host = Q.load_store(p).device_store()
    dev = Q.load_device_store(p)
    assert dev.config_hash == "0" * 64 and (dev.n_bits, dev.b_min) == (n_bits, b_min)
    ds = dev.device_store()
    for i, lid in enumerate(store.ordered_ids()):
        assert ds.shapes[i] == store.layers[lid].shape
        x = rng.standard_normal(store.layers[lid].shape[1]).astype(np.float32)
        for b in range(b_min, n_bits + 1):
            assert ds.layer_bytes(i, b) == host.layer_bytes(i, b)
            a, h = ds.dequantize(i, b).cpu().numpy(), host.dequantize(i, b).cpu().numpy()
            assert np.array_equal(a, h)
            assert np.array_equal(a, Q.dequantize(store.layers[lid], b))
            xt = torch.from_numpy(x)
            assert torch.equal(ds.gemv(i, b, xt), host.gemv(i, b, xt))


def test_bad_files_rejected(tmp_path):
    """Header checks run on the host before any device work (CPU test)."""
    p = str(tmp_path / "bad.dpqs")
    with open(p, "wb") as f:
        f.write(b"NOPE" + bytes(80))
    with pytest.raises(Q.QuantError):
        Q.load_device_store(p)


@pytest.mark.gpu
def test_reference_store_file_decodes_identically(report_setup, tmp_path):
    """The reference's toy store (sha256 = the hash every shipped plan embeds)
    loaded device-only decodes exactly like the host-loaded store."""
    S = report_setup
    p = str(tmp_path / "toy.dpqs")
    Q.save_store(S.store, p)
    assert Q.file_hash(p) == S.store_hash
    dstore = Q.load_device_store(p)
    assert dstore.param_counts() == S.store.param_counts()
    plan = R.load_plan(plan_path("dp_t3.5"), S.store)
    prompt = S.tokens[:16]
    out_h, tr_h = R.decode(S.weights, S.store, plan, prompt, 24, store_hash=S.store_hash)
    out_d, tr_d = R.decode(S.weights, dstore, plan, prompt, 24, store_hash=S.store_hash)
    assert out_d == out_h
    assert [s.bits for s in tr_d.steps] == [s.bits for s in tr_h.steps]
    assert [s.effective_bits for s in tr_d.steps] == [s.effective_bits for s in tr_h.steps]
