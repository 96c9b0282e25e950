"""Debug: prefill + a few steps, engine vs per-op graph vs oracle, on small configs."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))), "tests"))
import numpy as np
from oracle import dpq_oracle as O
from paper_2508_06041_b200 import model as M, quant as Q, runtime as R, _lib

def run(cfg, n_bits=6, static_bit=5, steps=4, seed=0):
    w = M.init_model(seed, cfg)
    store = Q.quantize_model(w, n_bits, 3)
    bits = {l: static_bit for l in store.layers}
    plan = R.sentinel_static_plan(bits, store.param_counts(), float(static_bit))
    toks = np.arange(steps) + 3
    out = {}
    for name, kw in (("engine", {}), ("ops", {"use_persistent": False})):
        eng = R.DecodeEngine(w, store, plan, **kw)
        kind = _lib.load().dpq_session_is_persistent(eng._h)
        lg = [eng.step(int(t), dynamic=(i > 0)) for i, t in enumerate(toks)]
        out[name] = (kind, np.array(lg))
    eo = O.Engine(w, store.layers, plan.layers, plan.M)
    ref = np.array([eo.step(int(t), dynamic=(i > 0)) for i, t in enumerate(toks)])
    for name, (kind, lg) in out.items():
        err = np.abs(lg - ref).max(axis=1) / np.abs(ref).max()
        print(cfg, name, "kind", kind, "rel err per step", err)

run(M.ModelConfig(n_blocks=2, d_model=32, n_heads=4, d_ff=64, seq_cap=64))
run(M.ModelConfig(n_blocks=1, d_model=32, n_heads=4, d_ff=64, seq_cap=64))
run(M.ModelConfig(n_blocks=1, d_model=64, n_heads=4, d_ff=128, seq_cap=64))
run(M.ModelConfig(n_blocks=1, d_model=64, n_heads=8, d_ff=128, seq_cap=64))
run(M.ModelConfig(n_blocks=1, d_model=32, n_heads=2, d_ff=64, seq_cap=64))
run(M.ModelConfig(n_blocks=1, d_model=128, n_heads=4, d_ff=64, seq_cap=64))
