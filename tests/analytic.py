"""Analytic expectations of the infinite-medium check problem (kind INFINITE:
one nuclide with energy-independent cross sections, density 1 atom/(b cm),
reflective box, every region the same fissionable material).

These hold for ANY correct analog Monte Carlo of that medium, so they pin both
the oracle and the GPU path against physics rather than against each other:
  * k_inf = nu*Sigma_f / Sigma_a (collision and track-length estimators: in
    expectation; absorption estimator: exactly, every history scores it once);
  * every history ends absorbed (no leakage in an infinite medium);
  * collisions per history ~ Geometric(p = Sigma_a/Sigma_t): mean Sigma_t/Sigma_a,
    variance (1-p)/p^2;
  * track length per history ~ Exponential(Sigma_a) (a geometric sum of
    Exp(Sigma_t) flights): mean 1/Sigma_a, variance 1/Sigma_a^2; the absorption
    rate tally (track x Sigma_a) has mean 1 per history.
"""
import math

import numpy as np

SIGMA_T, SIGMA_A, SIGMA_F, NU = 1.0, 0.4, 0.25, 2.5
K_INF = NU * SIGMA_F / SIGMA_A  # 1.5625
TALLY_SCALE = 2.0 ** 28


def check(res, tally, n, batches, inactive, nsigma=3.0):
    """Assert the analytic expectations on one run (oracle or GPU result
    structs: k_* per batch, n_events, n_absorbed/n_leaked/n_lost; tally =
    int64 fixed point [flux, absorption, fission, nu-fission] summed over
    active batches)."""
    kc = np.array([res.k_coll[b] for b in range(inactive, batches)])
    kt = np.array([res.k_track[b] for b in range(inactive, batches)])
    ka = np.array([res.k_abs[b] for b in range(batches)])
    # absorption estimator: K_INF per history exactly (fixed-point rounding only)
    assert np.all(np.abs(ka - K_INF) < 1e-6), ka
    for est in (kc, kt):
        sem = est.std(ddof=1) / math.sqrt(len(est))
        assert abs(est.mean() - K_INF) < nsigma * sem + 1e-12, (est.mean(), sem)
    h = n * batches
    assert res.n_absorbed == h and res.n_leaked == 0 and res.n_lost == 0
    p = SIGMA_A / SIGMA_T
    coll = res.n_events[3] / h
    assert abs(coll - 1.0 / p) < nsigma * math.sqrt((1.0 - p) / p ** 2 / h), coll
    ha = n * (batches - inactive)
    flux, absr = tally[0] / TALLY_SCALE / ha, tally[1] / TALLY_SCALE / ha
    assert abs(flux - 1.0 / SIGMA_A) < nsigma * (1.0 / SIGMA_A) / math.sqrt(ha), flux
    assert abs(absr - 1.0) < nsigma / math.sqrt(ha), absr
    fis, nufis = tally[2] / TALLY_SCALE, tally[3] / TALLY_SCALE
    assert abs(nufis / fis - NU) < 1e-6
    return {"k_coll": float(kc.mean()), "k_track": float(kt.mean()), "collisions_per_history": coll,
            "flux_per_history": flux}
