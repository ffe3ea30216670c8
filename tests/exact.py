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


def exact_mean_cuda(u) -> float:
    """exact_mean of a CUDA f64 tensor (the BASELINE-size sample sets): the same
    per-exponent integer sums, with torch on the device for the bulk."""
    import torch

    n = u.numel()
    m, e = torch.frexp(u)
    mi = torch.ldexp(m, torch.tensor(53.0, device=u.device, dtype=torch.float64)).to(torch.int64)
    e2 = e.to(torch.int64) - 53
    total = Fraction(0)
    for ev in torch.unique(e2).tolist():
        sel = mi[e2 == ev]
        pad = (-sel.numel()) % 512
        if pad:
            sel = torch.cat([sel, torch.zeros(pad, dtype=torch.int64, device=u.device)])
        parts = sel.view(-1, 512).sum(dim=1).cpu().numpy()
        total += Fraction(int(sum(int(x) for x in parts))) * Fraction(2) ** int(ev)
    return float(total / n)
