import os, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
from oracle import dpq_oracle as O
from paper_2508_06041_b200 import model as M, quant as Q, runtime as R, _lib
G = os.path.join(ROOT, "tests", "golden")
gs = json.load(open(os.path.join(G, "toy_summary.json")))
cfg = M.ModelConfig.from_dict(gs["config"])
w = M.init_model(gs["seed"], cfg)
store = Q.quantize_model(w, gs["n_bits"], gs["b_min"])
plan = R.load_plan(os.path.join(G, "plans", "dp_t3.5.json"), store)
toks = np.arange(6) + 40
for variant in ("plan", "static6", "static5"):
    if variant == "plan":
        pl = plan
    else:
        b = int(variant[-1])
        pl = R.sentinel_static_plan({l: b for l in store.layers}, store.param_counts(), float(b))
    res = {}
    for name, kw in (("engine", {}), ("ops", {"use_persistent": False})):
        eng = R.DecodeEngine(w, store, pl, g_dtype="f32", **kw)
        res[name] = np.array([eng.step(int(t), dynamic=False) for t in toks])
    eo = O.Engine(w, store.layers, pl.layers, pl.M)
    ref = np.array([eo.step(int(t), dynamic=False) for t in toks])
    for name, lg in res.items():
        print(variant, name, np.abs(lg - ref).max(axis=1) / np.abs(ref).max())
print(cfg)
print([(l.name, plan.layers[l].prefill_bit, plan.layers[l].pair) for l in store.ordered_ids()])
