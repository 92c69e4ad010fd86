"""Scenario inputs restated from reference batch.py -- TEST INFRASTRUCTURE ONLY."""

from __future__ import annotations

import numpy as np


def multipliers(seed: int, count: int, n: int, spread: float = 0.2, start: int = 0) -> np.ndarray:
    """Row i: (1-spread) + 2 spread U, U = first n doubles of
    Generator(Philox(key=[seed, i])) (batch.py:45-60)."""
    out = np.empty((count, n))
    for r in range(count):
        g = np.random.Generator(np.random.Philox(key=np.array([seed, start + r], dtype=np.uint64)))
        out[r] = (1.0 - spread) + 2.0 * spread * g.random(n)
    return out


def tx_specs(p_load, q_load, p_gen, q_gen, load_elements, theta_block, q_block, mult):
    """p_spec/q_spec rows for multiplier rows (batch.py:121-145)."""
    rows_p, rows_q = [], []
    for m in mult:
        p, q = p_load.copy(), q_load.copy()
        p[load_elements] *= m
        q[load_elements] *= m
        rows_p.append((p_gen - p)[theta_block])
        rows_q.append((q_gen - q)[q_block])
    return np.array(rows_p), np.array(rows_q)


def dist_specs(wye_s, delta_s, kinds, mult):
    """s_wye/s_delta rows (batch.py:146-151)."""
    kinds = np.array(kinds)
    return (np.array([wye_s * m[kinds == "wye"] for m in mult]),
            np.array([delta_s * m[kinds == "delta"] for m in mult]))
