"""Learning-rate schedule of PAPER.md §"Learning rate schedule" (:106-121).

Eq. 3 (:111):  lambda_i = lambda_0 * gamma^i          (i = epoch)
Eq. 4 (:117):  lambda_0(N, n) = lambda_0 / (1 + N/n)  (n = workers at which it halves, :119)
Clip (:121):   the effective base rate lambda_0 * N is clipped at 0.1.

Reading: the clip applies to the
reduced base rate before the per-epoch decay:
    lambda_0' = lambda_0 / (1 + N/n);  if lambda_0' * N > 0.1: lambda_0' = 0.1 / N
    lambda_e  = lambda_0' * gamma^e
"""
from __future__ import annotations


def base_rate(lambda0: float, N: int, n_half: float, max_eff: float = 0.1) -> float:
    lam = lambda0 / (1.0 + N / n_half)          # Eq. 4
    if lam * N > max_eff:                       # clip
        lam = max_eff / N
    return lam


def rate_for_epoch(lambda0: float, N: int, n_half: float, gamma: float, epoch: int,
                   max_eff: float = 0.1) -> float:
    return base_rate(lambda0, N, n_half, max_eff) * gamma ** epoch   # Eq. 3
