import os, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
from oracle import dpq_oracle as O
from paper_2508_06041_b200 import model as M, quant as Q, runtime as R, _lib
cfg = M.ModelConfig(n_blocks=1, d_model=32, n_heads=4, d_ff=64, seq_cap=64)
w = M.init_model(0, cfg)
store = Q.quantize_model(w, 6, 3)
toks = np.arange(3) + 40
ids = store.ordered_ids()
pats = {
  "q5k5v6": {"q": 5, "k": 5, "v": 6, "o": 5, "up": 5, "gate": 5, "down": 5},
  "q6k5v5": {"q": 6, "k": 5, "v": 5, "o": 5, "up": 5, "gate": 5, "down": 5},
  "up4gate5": {"q": 5, "k": 5, "v": 5, "o": 5, "up": 4, "gate": 5, "down": 5},
  "o6": {"q": 5, "k": 5, "v": 5, "o": 6, "up": 5, "gate": 5, "down": 5},
  "down6": {"q": 5, "k": 5, "v": 5, "o": 5, "up": 5, "gate": 5, "down": 6},
}
for nm, pat in pats.items():
    bits = {l: pat[l.kind] for l in ids}
    pl = R.sentinel_static_plan(bits, store.param_counts(), 5.0)
    eng = R.DecodeEngine(w, store, pl)
    lg = np.array([eng.step(int(t), dynamic=False) for t in toks])
    eo = O.Engine(w, store.layers, pl.layers, pl.M)
    ref = np.array([eo.step(int(t), dynamic=False) for t in toks])
    print(nm, np.abs(lg - ref).max(axis=1) / np.abs(ref).max(), flush=True)
