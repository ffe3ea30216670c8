"""Exact arithmetic helpers for the parity tests (test infrastructure)."""
from fractions import Fraction

import numpy as np


def exact_mean(samples) -> float:
    """The correctly rounded mean of f64 samples: every sample is m * 2^e with
    an integer m < 2^53, so the sum is exact in Python integers (per exponent,
    int64 partial sums of 512 mantissas, then arbitrary precision); float() of
    the Fraction rounds once.  colo's fleet statistics compute the mean as
    this value (exact fixed-point sum, divided once); the reference's finalize
    sums the sorted samples sequentially, which drifts from it by its own
    rounding (about n * eps relative at worst)."""
    u = np.ascontiguousarray(samples, np.float64)
    if not len(u):
        raise ValueError("exact_mean of no samples")
    m, e = np.frexp(u)
    mi = np.ldexp(m, 53).astype(np.int64)  # u == mi * 2^(e - 53), exactly
    e2 = e.astype(np.int64) - 53
    total = Fraction(0)
    for ev in np.unique(e2):
        sel = mi[e2 == ev]
        pad = (-len(sel)) % 512
        parts = np.pad(sel, (0, pad)).reshape(-1, 512).sum(axis=1)  # each < 512 * 2^53 = 2^62
        total += Fraction(int(sum(int(x) for x in parts))) * Fraction(2) ** int(ev)
    return float(total / len(u))


def exact_mean_cuda(u, chunk: int = 1 << 28) -> float:
    """exact_mean of a CUDA f64 tensor (the BASELINE-size sample sets): the same
    per-exponent integer sums, with torch on the device for the bulk, in chunks
    of `chunk` samples so the temporaries stay a few GB."""
    import torch

    n = u.numel()
    if not n:
        raise ValueError("exact_mean of no samples")
    sums = {}
    two53 = torch.tensor(53.0, device=u.device, dtype=torch.float64)
    for c0 in range(0, n, chunk):
        x = u[c0:c0 + chunk]
        m, e = torch.frexp(x)
        mi = torch.ldexp(m, two53).to(torch.int64)
        del m
        e2 = e.to(torch.int64) - 53
        del e
        for ev in torch.unique(e2).tolist():
            sel = mi[e2 == ev]
            pad = (-sel.numel()) % 512
            if pad:
                sel = torch.cat([sel, torch.zeros(pad, dtype=torch.int64, device=u.device)])
            parts = sel.view(-1, 512).sum(dim=1).cpu().numpy()
            sums[ev] = sums.get(ev, 0) + int(sum(int(x) for x in parts))
        del mi, e2
    total = sum((Fraction(v) * Fraction(2) ** int(ev) for ev, v in sums.items()), Fraction(0))
    return float(total / n)


def is_nearest_rank(u, q: float, v: float) -> bool:
    """v is the nearest-rank q-quantile of the CUDA f64 tensor u (metrics.hpp:48-53:
    sorted[ceil(q n) - 1]) without sorting: #(u < v) <= idx < #(u <= v)."""
    import math

    n = u.numel()
    idx = max(1, math.ceil(q * n)) - 1
    below = int((u < v).sum().item())
    at_or_below = int((u <= v).sum().item())
    return below <= idx < at_or_below
