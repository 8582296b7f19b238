"""TEST INFRASTRUCTURE ONLY — fp64 numpy restatement of the device CPD-ALS.

The reference has no ALS (SPEC.md:13 puts it out of scope; the only hook is the chaining
flag of mttkrp_all_modes, kernel.hpp:171-197), so this oracle is "parity unpinned" against
the reference: it restates standard CP-ALS (Kolda & Bader 2009) exactly as
DESIGN.md §6 specifies it for the device path:

  per mode d:  M = MTTKRP_d(current factors)         (chained: earlier modes already updated)
               V = ⊛_{w≠d} Y_wᵀ Y_w
               Y_d = M V⁻¹   (Cholesky; pseudo-inverse with 1e-12·λmax cut-off if not SPD)
               λ_r = ||Y_d[:, r]||₂ (1 when zero);  Y_d[:, r] /= λ_r
  fit = 1 - sqrt(max(0, ||X||² - 2⟨X,X̂⟩ + ||X̂||²)) / ||X||
"""
import numpy as np


def mttkrp64(dims, coords, values, factors, d):
    coords = np.asarray(coords).reshape(-1, len(dims))
    rank = factors[0].shape[1]
    term = np.repeat(np.asarray(values, np.float64)[:, None], rank, axis=1)
    for w in range(len(dims)):
        if w != d:
            term = term * np.asarray(factors[w], np.float64)[coords[:, w]]
    out = np.zeros((dims[d], rank), np.float64)
    np.add.at(out, coords[:, d], term)
    return out


def solve_inverse(V):
    try:
        L = np.linalg.cholesky(V)
        # same pivot rule as the device: a pivot <= 1e-12 * max diag(V) means "not SPD"
        if np.min(np.diag(L)) ** 2 <= 1e-12 * np.max(np.diag(V)):
            raise np.linalg.LinAlgError("near-singular")
        Linv = np.linalg.inv(L)
        return Linv.T @ Linv
    except np.linalg.LinAlgError:
        lam, W = np.linalg.eigh(V)
        keep = np.abs(lam) > 1e-12 * np.abs(lam).max()
        return (W[:, keep] / lam[keep]) @ W[:, keep].T


def als_iteration(dims, coords, values, factors):
    """One iteration; returns (new factors, lambda, fit, M of the last mode)."""
    Y = [np.asarray(f, np.float64).copy() for f in factors]
    n = len(dims)
    grams = [y.T @ y for y in Y]
    lam = np.ones(Y[0].shape[1])
    M = None
    for d in range(n):
        M = mttkrp64(dims, coords, values, Y, d)
        V = np.ones_like(grams[0])
        for w in range(n):
            if w != d:
                V = V * grams[w]
        Y[d] = M @ solve_inverse(V)
        lam = np.sqrt(np.maximum((Y[d] ** 2).sum(axis=0), 0.0))
        lam[lam == 0] = 1.0
        Y[d] = Y[d] / lam
        grams[d] = Y[d].T @ Y[d]
    norm2 = float(np.sum(np.asarray(values, np.float64) ** 2))
    inner = float(np.sum(M * Y[n - 1] * lam))
    H = np.ones_like(grams[0])
    for g in grams:
        H = H * g
    model2 = float(lam @ H @ lam)
    fit = 1.0 - np.sqrt(max(0.0, norm2 - 2 * inner + model2)) / np.sqrt(norm2)
    return Y, lam, fit, M
