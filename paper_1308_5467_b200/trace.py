"""Hutchinson trace estimation (specdens/stochastic.py:77-108) on the device.

Tr A ~ mean_l v_l^T A v_l.  The quadratic forms are the first Chebyshev moment
of the unmapped operator (B = A, c = 0, d = 1: the step epilogue's (y - 0 x)/1
is y exactly), so one step of the fused moment kernel over the whole probe
block gives every v_l^T A v_l; mean and unbiased variance on the device.
"""

from dataclasses import dataclass

from . import _native
from . import engine as E


@dataclass(frozen=True)
class TraceEstimate:
    """Stochastic trace estimate with its sample statistics (stochastic.py:77-94)."""

    value: float
    n_samples: int
    sample_variance: float

    def __post_init__(self):
        if self.n_samples < 1:
            raise ValueError("a trace estimate needs at least one sample")
        if self.sample_variance < 0.0:
            raise ValueError("sample variance cannot be negative")


def estimate_trace_quadratic(op, source, n_vec, threads=None, device=None):
    """Hutchinson estimate of Tr A: the average of v^T (A v) over probes (stochastic.py:97-108)."""
    if n_vec < 1:
        raise ValueError("need at least one probe vector")
    torch = E._torch()
    run = E.run_chebyshev(op, 1, source, n_vec, _native.SDB_CHEB_DIRECT, device=device)
    with torch.cuda.device(run.zeta_pp.device):
        terms = run.zeta_pp[:, 1]
        mean = terms.mean()
        var = terms.var(unbiased=True) if n_vec > 1 else torch.zeros_like(mean)
        packed = torch.stack([mean, var]).cpu().numpy()
    E.credit_counters(run.resolved, n_vec, 1)
    return TraceEstimate(value=float(packed[0]), n_samples=n_vec, sample_variance=float(packed[1]))
