"""A-priori fp32 error bounds for the toy-model kernels (softmax_grad, dynamic criterion) against exact arithmetic.

Test infrastructure (tolerances only: no expected value comes from here). The kernels evaluate the toy model's
gradient and the dynamic-criterion statistics (readings C18 and C26) in fp32 with fp64 accumulation of the
criterion sums; the oracle evaluates the same definitions in fp64. This module bounds the difference by first-order
rounding-error analysis of the kernels' written operation order (kernels.cu softmax_fwd / softmax_bwd /
criterion_partial / criterion_final), in the standard model fl(a op b) = (a op b)(1 + e), |e| <= u = 2^-24, with
gamma_k = k u / (1 - k u) for a sum whose every term passes through at most k roundings (Higham, Accuracy and
Stability of Numerical Algorithms, Lemma 3.1 / §4.2 -- valid for any summation order of that depth):

  logits     z_bc = sum_i x_bi W_ic: per-thread FMA chain (ceil(d/256) terms), 5 warp-shuffle levels, 8 warp partials
             -> |dz_bc| <= gamma_k sum_i |x_bi||W_ic|,  k = ceil(d/256) + 5 + 8
  softmax    p = expf(z - m) / sum_k expf(z_k - m): argument rounding u|z_c - m| (relative error of exp), expf <= 2 ulp
             <= 4u relative (CUDA math library), C-1 sequential adds for the denominator, one correctly rounded
             division; plus the propagated logit error dp_c = p_c (dz_c - sum_k p_k dz_k)
  residual   r_bc = p_bc / B for c != y (exact for B a power of two), r_by = -(sum_{c != y} p_bc) / B (C-2 adds)
  gradient   g_ic = sum_b X_bi r_bc, sequential FMA over b -> sum_b |X_bi| dr_bc + gamma_B sum_b |X_bi||r_bc|
  criterion  Delta = g - g_prev.  |Delta| from fp64 differences of the fp32 inputs: d|Delta| <= || dg + dg_prev ||_2.
             u_b = B x_b^T (Delta r_b) - Delta^T g with the per-sample Delta rounded once to fp32 (g[k] - g_prev[k]
             in fp32), everything after in fp64; sigma = ||u||_2 / (B |Delta|).
             => d sigma <= ||du||_2 / (B (|Delta| - d|Delta|)) + sigma d|Delta| / (|Delta| - d|Delta|)

The cancellation factor of the criterion is explicit: the absolute errors dg and dg_prev scale with |g| and
|g_prev|, while |Delta| = |g - g_prev| can be much smaller, so the relative error of |Delta| and sigma grows as
(|g| + |g_prev|) / |Delta|. The bounds are first order; they are multiplied by 1.01 to cover the dropped O(u^2)
terms, and the final fp32 casts of the two statistics add u relative each.
"""
from __future__ import annotations

import math

import numpy as np

U = 2.0 ** -24          # fp32 unit roundoff
U64 = 2.0 ** -53        # fp64 unit roundoff
SAFETY = 1.01           # covers the dropped second-order terms


def gamma(k: int, u: float = U) -> float:
    return k * u / (1.0 - k * u)


def softmax_grad_bounds(X, y, W, threads: int = 256):
    """Exact (fp64) logits, probabilities, residuals r = (p - onehot(y)) / B and gradient g = X^T r of the softmax
    regression at W (d x C, row-major flat), with elementwise bounds Er (B x C) and Eg (d*C) on the fp32 kernel's
    deviation from them. Returns dict(z, p, r, g, Er, Eg)."""
    X = np.asarray(X, np.float64)
    y = np.asarray(y, np.int64)
    B, d = X.shape
    Wm = np.asarray(W, np.float64).reshape(d, -1)
    C = Wm.shape[1]
    z = X @ Wm
    dz = gamma(math.ceil(d / threads) + 5 + 8) * (np.abs(X) @ np.abs(Wm))
    m = z.max(axis=1, keepdims=True)
    e = np.exp(z - m)
    p = e / e.sum(axis=1, keepdims=True)
    rel_e = 4 * U + U * np.abs(z - m)                                  # expf argument rounding + 2 ulp
    rel_p = (dz + (p * dz).sum(axis=1, keepdims=True)                  # propagated logit error
             + rel_e + rel_e.max(axis=1, keepdims=True) + gamma(max(C - 1, 0)) + U)
    Ep = p * rel_p
    pow2 = B & (B - 1) == 0
    onehot = np.zeros_like(p)
    onehot[np.arange(B), y] = 1.0
    r = (p - onehot) / B
    Er = Ep / B + (0.0 if pow2 else U * np.abs(r))
    for b in range(B):                                                 # true class: -(sum of the others) / B
        others = np.arange(C) != y[b]
        Er[b, y[b]] = (Ep[b, others].sum() + gamma(max(C - 2, 0)) * p[b, others].sum()) / B \
            + (0.0 if pow2 else U * abs(r[b, y[b]]))
    g = X.T @ r
    Eg = np.abs(X).T @ Er + gamma(B) * (np.abs(X).T @ np.abs(r))
    return dict(z=z, p=p, r=r, g=g.ravel(), Er=Er, Eg=SAFETY * Eg.ravel())


def criterion_bounds(X, y, W, g_prev, Eg_prev):
    """Bounds on the criterion kernel's (|Delta|, sigma) against the exact values at W with the exact previous batch
    gradient g_prev, when the kernel is handed a g_prev within Eg_prev (elementwise) of it.
    Returns (nd, sigma, d_nd, d_sigma, Eg) with nd, sigma computed here in fp64 (for the band only)."""
    X = np.asarray(X, np.float64)
    B, d = X.shape
    s = softmax_grad_bounds(X, y, W)
    g, Eg, r, Er = s["g"], s["Eg"], s["r"], s["Er"]
    C = r.shape[1]
    gp = np.asarray(g_prev, np.float64)
    Egp = np.asarray(Eg_prev, np.float64)
    delta = g - gp
    nd = float(np.linalg.norm(delta))
    # |Delta|: fp64 differences of the two fp32 vectors, fp64 sum of squares and sqrt, then the fp32 cast
    dd = Eg + Egp
    d_nd = float(np.linalg.norm(dd)) + gamma(d * C + 2, U64) * nd + U * nd
    # per-sample terms: Delta rounded once to fp32, then fp64
    dd_b = dd + U * (np.abs(delta) + dd)
    Dm, dDm = delta.reshape(d, C), dd_b.reshape(d, C)
    part = B * np.einsum("bi,ic,bc->b", X, Dm, r)
    abs_terms = B * np.einsum("bi,ic,bc->b", np.abs(X), np.abs(Dm), np.abs(r))
    d_part = B * (np.einsum("bi,ic,bc->b", np.abs(X), dDm, np.abs(r))
                  + np.einsum("bi,ic,bc->b", np.abs(X), np.abs(Dm), Er)) + gamma(d * C + 8, U64) * abs_terms
    dg = float(delta @ g)
    d_dg = float(dd @ np.abs(g) + np.abs(delta) @ Eg) + gamma(d * C + 2, U64) * float(np.abs(delta) @ np.abs(g))
    ub = part - dg
    d_ub = d_part + d_dg + gamma(2, U64) * np.abs(ub)
    sigma = float(np.linalg.norm(ub) / (B * nd)) if nd > 0 else 0.0
    if nd > 0 and d_nd < nd:
        d_sigma = (float(np.linalg.norm(d_ub)) / (B * (nd - d_nd)) + sigma * d_nd / (nd - d_nd)) * SAFETY + U * sigma
    else:
        d_sigma = math.inf        # |Delta| not resolved at fp32: sigma is not determined
    return nd, sigma, SAFETY * d_nd, d_sigma, Eg
