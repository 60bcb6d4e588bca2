"""CPU check of the algebra behind k_slices3's small-slice A system (no GPU).

The reference solves A u = s o xv with A = vtv o s s^T + sh I by Cholesky
(`src/_kernels.py:86-100` of the reference).  The kernel uses
A = S (vtv + diag(d)) S, d_r = sh / s_r^2, and the Neumann series of
(vtv + diag(d))^{-1} around P = vtv^{-1}: first order when
rho = max_r d_r * ||P||_inf <= 1e-6, second order when rho <= 1e-4, the exact
sweep otherwise (dash_slices3.cuh).  This test restates that selection rule in
numpy and checks the truncation bound against a direct solve over weights
spread across many magnitudes, with the J=128, R=16 shape of the large config.
"""
import numpy as np

RIDGE_EPS = 1e-10
RHO1, RHO2 = 1e-6, 1e-4


def _neumann_u(vtv, s, xv):
    R = len(s)
    sh = RIDGE_EPS * np.sum(np.diag(vtv) * s * s) / R
    P = np.linalg.inv(vtv)
    d = sh / (s * s)
    rho = d.max() * np.abs(P).sum(axis=1).max()
    if not rho <= RHO2:
        return None, rho
    y = xv @ P                        # rows y_i = P xv_i (P symmetric)
    c1 = (y * d) @ P                  # P d y
    u = y - c1
    if rho > RHO1:
        u = u + (c1 * d) @ P          # + P d P d y
    return u / s, rho


def _direct_u(vtv, s, xv):
    R = len(s)
    sh = RIDGE_EPS * np.sum(np.diag(vtv) * s * s) / R
    A = vtv * np.outer(s, s) + sh * np.eye(R)
    return np.linalg.solve(A, (xv * s).T).T


def test_neumann_series_matches_direct_solve_within_the_stated_bound():
    rng = np.random.default_rng(3)
    J, R = 128, 16
    V = rng.uniform(size=(J, R))
    vtv = V.T @ V
    taken = {"first": 0, "second": 0, "sweep": 0}
    unscaled_fast = 0
    for trial in range(400):
        s = rng.uniform(size=R)
        k = trial % 8
        if k:  # spread magnitudes: 1e-1 .. 1e-7 on a couple of entries
            cols = rng.choice(R, size=2, replace=False)
            s[cols] *= 10.0 ** -k
            if trial % 5 == 0:
                s[cols[0]] *= -1.0
        xv = rng.normal(size=(rng.integers(1, 9), R))
        u, rho = _neumann_u(vtv, s, xv)
        if u is None:
            taken["sweep"] += 1
            continue
        taken["first" if rho <= RHO1 else "second"] += 1
        unscaled_fast += k == 0
        ref = _direct_u(vtv, s, xv)
        err = np.abs(u - ref).max() / np.abs(ref).max()
        # truncation (rho^2 or rho^3 <= 1e-12) plus rounding of the two routes
        assert err < 1e-9, (trial, rho, err)
    # all three branches are exercised by this spread
    assert min(taken.values()) > 0, taken
    assert unscaled_fast >= 45, unscaled_fast  # U[0,1] weights (the planted workload): nearly all fast


def test_zero_weight_forces_the_exact_path():
    rng = np.random.default_rng(5)
    V = rng.uniform(size=(64, 8))
    s = rng.uniform(size=8)
    s[3] = 0.0
    with np.errstate(divide="ignore"):
        u, rho = _neumann_u(V.T @ V, s, rng.normal(size=(3, 8)))
    assert u is None and not np.isfinite(rho)
