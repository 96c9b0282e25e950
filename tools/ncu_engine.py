"""Short engine run for ncu: 8B-shaped model, DP plan, prefill + one
decode_greedy(4) launch (the profiled engine_kernel launch is the last one).

    ncu ... python tools/ncu_engine.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench as B  # noqa: E402
from paper_2508_06041_b200 import runtime as R, synth  # noqa: E402

torch.cuda.set_device(0)
cfg, n_bits, b_min = B.model_config("llama3_8b")
w, store, _ = synth.random_device_model(cfg, n_bits, b_min, seed=1234)
pairs, prefill, high = B.pairs_for_target(store, 3.5)
plan = synth.projection_plan(store, pairs, prefill, k=64, seed=0, target=3.5)
synth.calibrate_thresholds(w, store, plan, np.random.default_rng(7).integers(0, cfg.vocab, 8), high_rate=high)
eng = R.DecodeEngine(w, store, plan, g_dtype="f16")
eng.prefill(np.random.default_rng(11).integers(0, cfg.vocab, 4))
torch.cuda.synchronize()
torch.cuda.profiler.start()          # ncu --profile-from-start off: only this launch
eng.decode_greedy(4)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("steps", len(eng.trace.steps), "eff bits", eng.trace.steps[-1].effective_bits)
