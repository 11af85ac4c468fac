"""Seeded synthetic inputs shared by the oracle side (tests, bench cpu_baseline) and the CUDA side (tests, bench).

Holds NONE of the method's arithmetic: only data the workers would have read (a toy classification dataset and
its mini-batch order) and the configuration geometry of BASELINE.json's configs. Gradients and arrival schedules are
NOT generated here: each side implements the counter-based generators of SURVEY.md §8d independently.
"""
from __future__ import annotations

import numpy as np

GRAD_SEED = 20241018      # SURVEY §8d gradient seed
SCHED_SEED = 7            # SURVEY §8d schedule seed

# BASELINE.json configs (SURVEY §8 geometry table)
RESNET32_P = 464_154      # ResNet-32 / CIFAR-10 shaped (computed in SURVEY §8; the paper prints no count)
RESNET50_P = 25_557_032   # ResNet-50 shaped (torchvision, BASELINE.json "25.6M")


def toy_dataset(seed: int = 1, n_points: int = 1000, d: int = 1024, C: int = 8, mean_scale: float = 0.5,
                feature_scale: float = 1.0):
    """A Gaussian mixture of C classes in d-1 dims plus a constant-1 bias feature (P = d*C).
    Class means ~ N(0, I) scaled by `mean_scale` (0.5: separable; 0.05: overlapping classes, the gradient noise never
    vanishes), unit-variance noise; labels uniform; the d-1 features are multiplied by `feature_scale`.
    Returns X float32 [N, d], y int32."""
    rng = np.random.Generator(np.random.PCG64(seed))
    means = rng.standard_normal((C, d - 1)) * mean_scale
    y = rng.integers(0, C, n_points).astype(np.int32)
    X = (means[y] + rng.standard_normal((n_points, d - 1))) * feature_scale
    X = np.concatenate([X, np.ones((n_points, 1))], axis=1).astype(np.float32)
    return X, y


# Config 1 (BASELINE configs[0]; SURVEY §8(d) toy data): 1,000 training points, plus 1,000 held-out points from the same
# mixture for test accuracy. Features scaled by 1/32 (|x| ~ 1, so the paper's eta = 0.1 is a stable step for softmax
# regression) and class means at 0.2: the classes overlap, so the loss is still falling when training switches from
# BSP to ASP at 50% (ln 8 = 2.079 -> ~1.95 at the switch -> ~1.77 after the ASP phase, oracle run).
TOY_RECIPE = dict(seed=1, n_points=2000, mean_scale=0.2, feature_scale=1.0 / 32)


def toy_split():
    """Config-1 data: (X_train [1000, 1024], y_train, X_test [1000, 1024], y_test)."""
    X, y = toy_dataset(**TOY_RECIPE)
    return X[:1000], y[:1000], X[1000:], y[1000:]


def minibatch_order(seed: int, n_points: int, n_batches: int, B: int) -> np.ndarray:
    """Sequential mini-batches over a seed-shuffled permutation, reshuffled each epoch. [n_batches, B]."""
    rng = np.random.Generator(np.random.PCG64(seed + 1))
    out = []
    perm = rng.permutation(n_points)
    pos = 0
    for _ in range(n_batches):
        if pos + B > n_points:
            perm = rng.permutation(n_points)
            pos = 0
        out.append(perm[pos:pos + B])
        pos += B
    return np.stack(out).astype(np.int64)
