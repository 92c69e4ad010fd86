"""Algorithmic work per scenario, the numerators of the reported rooflines.

Pinned to SURVEY.md 8(d) so that the count cannot be gamed by the ordering
or the kernel design:

* NR (HBM-bound): bytes = K*8*(2*nnz_LU + 2n + 3n_J) + 8*(2n + 2n_J), with
  nnz_LU the MMD(A^T+A) static-pivot factor size (74,280 for gb2224,
  1,777 for case118) whatever ordering the engine uses; K = Newton
  iterations the scenario actually returned.
* Z-Bus (FP64-tensor-bound): flops = (K+1)*(8*n*|l| + 4n + 20*n_loads),
  K iterations plus the residual certificate; dense 8n^2 counting is not
  allowed.
"""

from __future__ import annotations

import numpy as np

PINNED_NNZ_LU = {2224: 74280, 118: 1777}


def nr_bytes_per_scenario(iterations, n_bus: int, n_j: int, nnz_lu: int) -> np.ndarray:
    nnz = PINNED_NNZ_LU.get(n_bus, nnz_lu)
    k = np.asarray(iterations, dtype=np.float64)
    return k * 8.0 * (2 * nnz + 2 * n_bus + 3 * n_j) + 8.0 * (2 * n_bus + 2 * n_j)


def nr_bytes_per_scenario_executed(iterations, n_bus: int, n_j: int, nnz_lu: int) -> np.ndarray:
    """As nr_bytes_per_scenario, but the first Newton step solves with the
    flat-start LU shared by every scenario (nr_flat_start_factor), so it moves
    no per-scenario factor: K-1 factor passes plus the step-0 vectors."""
    nnz = PINNED_NNZ_LU.get(n_bus, nnz_lu)
    k = np.asarray(iterations, dtype=np.float64)
    kf = np.maximum(k - 1.0, 0.0)
    step0 = np.where(k > 0, 8.0 * (2 * n_bus + 3 * n_j), 0.0)
    return kf * 8.0 * (2 * nnz + 2 * n_bus + 3 * n_j) + step0 + 8.0 * (2 * n_bus + 2 * n_j)


def zbus_flops_per_scenario(iterations, n: int, n_l: int, n_loads: int) -> np.ndarray:
    k = np.asarray(iterations, dtype=np.float64)
    return (k + 1) * (8.0 * n * n_l + 4.0 * n + 20.0 * n_loads)


def zbus_bytes_per_scenario(n: int, n_loads: int) -> float:
    return 16.0 * n_loads + 16.0 * n + 32.0
