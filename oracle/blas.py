"""Batched fp64 kernel module -- TEST INFRASTRUCTURE ONLY (the parity oracle).

A restatement of the reference's numpy backend (`_kernels_numpy.py:19-58`, selected by
`backend.py:18-34` with PARAQ_BACKEND=numpy) with one change: ``affine_rows`` computes
all rows in one BLAS product instead of one ``w @ x[r] + b`` per row.  The result
differs from the per-row loop only in fp64 summation order -- the reference itself
accepts that between its two backends (rtol 1e-12 on Q, 1e-10 on gradients,
`pkg/tests/test_backend.py:59-63`).  It exists so the oracle can run the Nature-CNN at
batch 1024 / W 512 in seconds; `oracle/_lib.py` (kernels.c) stays the bit-exact module
pinned to the golden vectors.
"""

from __future__ import annotations

import numpy as np

BACKEND_NAME = "oracle-blas"


def affine_rows(w, b, x):
    """_kernels_numpy.py:19-23 (batched)."""
    return np.asarray(x, dtype=np.float64) @ np.asarray(w, dtype=np.float64).T + b


def relu(x):
    """_kernels_numpy.py:26-27."""
    return np.maximum(x, 0.0)


def output_delta(q, actions, targets):
    """_kernels_numpy.py:30-35: (q[a] - target) / n at the taken action, 0 elsewhere."""
    n = q.shape[0]
    delta = np.zeros_like(q)
    rows = np.arange(n)
    delta[rows, actions] = (q[rows, actions] - targets) / n
    return delta


def weight_grad(delta, acts):
    """_kernels_numpy.py:38-39."""
    return delta.T @ acts


def bias_grad(delta):
    """_kernels_numpy.py:42-43."""
    return delta.sum(axis=0)


def hidden_delta(delta, w, pre):
    """_kernels_numpy.py:46-47."""
    return (delta @ w) * (pre > 0.0)


def rmsprop_flat(p, g, m, v, lr, rho, kappa):
    """_kernels_numpy.py:50-54 (centered RMSProp, kappa inside the square root)."""
    m2 = rho * m + (1.0 - rho) * g
    v2 = rho * v + (1.0 - rho) * g * g
    p2 = p - lr * g / np.sqrt(v2 - m2 * m2 + kappa)
    return p2, m2, v2
