"""Synthetic request traces shaped like the paper's workloads (numbers only).

Prompt lengths ~ lognormal with mean 12035 tokens (Mooncake) and sigma 1.0, clipped to
[512, 32768]; output lengths ~ lognormal with mean 343 and sigma 1.0, clipped to [16, 2048]; bursty
arrivals: Gamma inter-arrival times with coefficient of variation 2 at `qps` requests per second.
"""
from __future__ import annotations

import numpy as np


def lognormal_mean(rng, mean: float, sigma: float, n: int) -> np.ndarray:
    mu = np.log(mean) - sigma * sigma / 2.0   # E[exp(N(mu, sigma^2))] = mean
    return rng.lognormal(mu, sigma, size=n)


def bursty_trace(n_req: int, qps: float, seed: int, isl_mean=12035.0, osl_mean=343.0, sigma=1.0, cv=2.0,
                 isl_clip=(512, 32768), osl_clip=(16, 2048)):
    """[(id, prompt_len, output_len, arrival_s)] with non-decreasing arrivals."""
    rng = np.random.Generator(np.random.PCG64(seed))
    k = 1.0 / (cv * cv)
    gaps = rng.gamma(k, 1.0 / (qps * k), size=n_req)
    t = np.cumsum(gaps) - gaps[0]
    isl = np.clip(lognormal_mean(rng, isl_mean, sigma, n_req), *isl_clip).astype(int)
    osl = np.clip(lognormal_mean(rng, osl_mean, sigma, n_req), *osl_clip).astype(int)
    return [(i, int(isl[i]), int(osl[i]), float(t[i])) for i in range(n_req)]
