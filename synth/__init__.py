"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NO arithmetic of the LS-SVM method: it only draws data.  It is the one
module both sides (``oracle/`` and ``paper_2202_12674_b200/``) may consume.

Recipe: the paper trains on scikit-learn
``make_classification`` "planes" data -- two adjacent clusters, 1 % random labels,
power-of-two shapes (§IV-B).  The generator script itself is not in the
paper, so the exact parameters are our reading (reading R-15):
n_informative=2, n_redundant=0, n_clusters_per_class=1, class_sep=1, flip_y=0.01,
hypercube=True.  Train and test come from ONE call so they share the cluster geometry.

Configs (BASELINE.json ``configs``, in order):
  C0  256 x 16     linear  fp64  eps 1e-10
  C1  2^14 x 2^10  RBF     fp64  gamma = 1/d   (bench.py default workload)
  C2  2^16 x 2^12  linear  fp64
  C3  2^15 x 2^11  poly    fp32  degree 3, gamma = 1/d, coef0 = 0
  C4  2^17 x 2^12  RBF     fp64  + predict on 2^15 test points
"""
from __future__ import annotations

import dataclasses
import hashlib

import numpy as np

SEED_BASE = 220212674  # + config index

LINEAR, POLYNOMIAL, RBF = 0, 1, 2


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    m: int
    d: int
    kernel: int
    dtype: str  # "f64" | "f32"
    gamma: float
    degree: int = 3
    coef0: float = 0.0
    C: float = 1.0
    eps: float = 1e-10
    n_test: int = 0
    index: int = 0


def configs() -> dict[str, Config]:
    return {
        "C0": Config("C0", 256, 16, LINEAR, "f64", 1.0 / 16, n_test=256, index=0),
        "C1": Config("C1", 2**14, 2**10, RBF, "f64", 2.0**-10, n_test=2**13, index=1),
        "C2": Config("C2", 2**16, 2**12, LINEAR, "f64", 2.0**-12, n_test=2**13, index=2),
        "C3": Config("C3", 2**15, 2**11, POLYNOMIAL, "f32", 2.0**-11, degree=3, coef0=0.0,
                     eps=1e-6, n_test=2**13, index=3),
        "C4": Config("C4", 2**17, 2**12, RBF, "f64", 2.0**-12, n_test=2**15, index=4),
    }


def planes(m: int, d: int, n_test: int = 0, seed: int = SEED_BASE, dtype=np.float64):
    """make_classification "planes".  Returns X[m,d], y[m] (+1/-1), Z[n_test,d], yz.

    X/Z are C-contiguous point-major (row = point).  For fp32 configs the values are rounded
    ONCE here; every consumer (oracle upcasts to fp64) sees the same rounded values.
    """
    from sklearn.datasets import make_classification

    X_all, y01 = make_classification(
        n_samples=m + n_test, n_features=d, n_informative=min(2, d), n_redundant=0,
        n_repeated=0, n_classes=2, n_clusters_per_class=1, class_sep=1.0, flip_y=0.01,
        hypercube=True, shift=0.0, scale=1.0, shuffle=True, random_state=seed)
    y_all = np.where(y01 == 1, 1.0, -1.0)
    X_all = np.ascontiguousarray(X_all.astype(dtype))
    y_all = y_all.astype(dtype)
    X, Z = np.ascontiguousarray(X_all[:m]), np.ascontiguousarray(X_all[m:])
    y, yz = y_all[:m].copy(), y_all[m:].copy()
    # both classes must be present; make_classification guarantees it for m>=16
    return X, y, Z, yz


def config_data(cfg: Config, m: int | None = None, d: int | None = None, n_test: int | None = None):
    """Data for a config, optionally at a reduced size (same recipe, same seed)."""
    dt = np.float32 if cfg.dtype == "f32" else np.float64
    return planes(m or cfg.m, d or cfg.d, cfg.n_test if n_test is None else n_test,
                  seed=SEED_BASE + cfg.index, dtype=dt)


def random_small(rng: np.random.Generator, m: int, d: int, dtype=np.float64):
    """Small random dense two-class instance (normal features, balanced random labels)."""
    X = rng.standard_normal((m, d)).astype(dtype)
    y = np.where(rng.random(m) < 0.5, 1.0, -1.0).astype(dtype)
    y[0], y[-1] = 1.0, -1.0  # both classes present
    return np.ascontiguousarray(X), y


def random_vector(rng: np.random.Generator, n: int, dtype=np.float64):
    return rng.standard_normal(n).astype(dtype)


def sha16(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]
