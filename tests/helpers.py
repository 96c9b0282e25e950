"""Shared test helpers: oracle runners and the parity rules.

Parity rule: decisions bit-exact except where the reference
estimate lies within eps*|T| of the threshold; after the first such tie the
comparison switches to forced-bits replay of the reference trace.
"""

from __future__ import annotations

import numpy as np

from oracle import dpq_oracle as O
from paper_2508_06041_b200 import model as M

EPS_DECISION = {"f32": 1e-4, "f16": 1e-3, "e4m3": 1e-2}


def oracle_engine(weights, store, plan, **kw):
    return O.Engine(weights, store.layers, plan.layers, plan.M, **kw)


def oracle_eval(weights, store, plan, tokens, **kw):
    eng = oracle_engine(weights, store, plan, **kw)
    ppl, losses = O.eval_perplexity(eng, tokens)
    return ppl, losses, eng


def canon(ids):
    return sorted(ids, key=lambda l: (l.block, M.KINDS.index(l.kind)))


def trace_arrays(records, ids):
    """bits / estimates (NaN = None) / exact as [steps][layers] arrays."""
    keyed = [O.key(l) for l in ids]

    def get(d, l, k):
        if l in d:
            return d[l]
        return d.get(k)

    bits = np.array([[get(r.bits, l, k) for l, k in zip(ids, keyed)] for r in records])
    est = np.array([[np.nan if get(r.estimates, l, k) is None else get(r.estimates, l, k)
                     for l, k in zip(ids, keyed)] for r in records], dtype=np.float64)
    return bits, est


def decision_mismatches(bits_dev, bits_ref, est_ref, T, eps, until_first=True):
    """Decisions that differ although |est_ref - T| > eps*|T|.

    Scanned in execution order (step-major, layers in block/kind order). With
    until_first (the free-run rule of SURVEY 8c) the scan stops at the first
    differing decision: later layers see a different input from there on, so
    only that first one is held to the eps rule.
    """
    bad = []
    for s in range(bits_ref.shape[0]):
        for i in range(bits_ref.shape[1]):
            if bits_dev[s, i] != bits_ref[s, i]:
                e, t = est_ref[s, i], T[i]
                if not (np.isfinite(e) and np.isfinite(t) and abs(e - t) <= eps * abs(t)):
                    bad.append((s, i, bits_dev[s, i], bits_ref[s, i], e, t))
                if until_first:
                    return bad
    return bad
