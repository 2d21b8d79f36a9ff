"""BASELINE.json configurations (C1-C5) and their input conventions.

Inputs follow einplan_run_json (capi.cpp:206-208): operand k of the einsum
gets random_tensor(shape, seed + k), seed 0.  C2 (the CP-ALS sweep) shares
one factor set across the three modes: X = seed 0, A/B/C = seeds 1/2/3
(SURVEY.md §8(d)).
"""
import numpy as np

import oracle

MT5 = "ijklm,ja,ka,la,ma->ia"

CONFIGS = {
    "C1": {"einsums": ["ijk,ja,ka->ia"], "procs": [1, 2, 4, 8],
           "extents": lambda P: dict(i=512, j=512, k=512, a=24)},
    "C2": {"einsums": ["ijk,ja,ka->ia", "ijk,ia,ka->ja", "ijk,ia,ja->ka"], "procs": [1, 2, 4, 8],
           "extents": lambda P: dict(i=1024, j=1024, k=1024, a=32)},
    "C3": {"einsums": [MT5], "procs": [1, 2, 4, 8],
           "extents": lambda P: dict(i=64, j=64, k=64, l=64, m=64, a=24)},
    "C4": {"einsums": ["ijk,jb,kc->ibc"], "procs": [1, 2, 4, 8],
           "extents": lambda P: dict(i=1024, j=1024, k=1024, b=64, c=64)},
    "C5": {"einsums": ["ijklm,jb,kc,ld,me->ibcde"], "procs": [1, 2, 4, 8],
           "extents": lambda P: dict(i=64 * P, j=64, k=64, l=64, m=64, b=16, c=16, d=16, e=16)},
}

# factor seed per mode letter for C2's shared factors
C2_FACTOR_SEED = {"i": 1, "j": 2, "k": 3}


def seeded(einsum, ext, seed=0):
    return oracle.seeded_inputs(einsum, ext, seed)


def c2_inputs(mode, ext):
    e = CONFIGS["C2"]["einsums"][mode]
    ins, _ = oracle.parse(e)
    ops = [oracle.random_tensor(oracle.shape_of(ins[0], ext), 0)]
    for t in ins[1:]:
        ops.append(oracle.random_tensor(oracle.shape_of(t, ext), C2_FACTOR_SEED[t[0]]))
    return ops
