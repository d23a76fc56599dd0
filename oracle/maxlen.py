"""Max inference length under an activation budget (test infrastructure only).

SPEC cmd_maxlen, the desk-scale analog of the paper's "11.7-fold
extension in the max inference length" for 1D inputs and "3.2-fold" for 2D
(§4.2): binary-search the largest sequence length whose (a) unchunked
Eq. 1 peak and (b) best chunk plan's Eq. 2 peak fit the budget.  Feasibility is
the planner's own: peak < budget, strict.  Lengths are searched on a grid
of `step` (128: whole tensor-core row tiles on the GPU).
"""
from __future__ import annotations

from .memory import profile
from .select import select
from .workloads import block


def _largest(fits, step: int, cap: int) -> int:
    """Largest multiple of `step` in [step, cap] with fits(N) true (fits monotone
    non-increasing in N); 0 when even `step` does not fit."""
    if not fits(step):
        return 0
    lo, hi = 1, 2
    while hi * step <= cap and fits(hi * step):
        lo, hi = hi, hi * 2
    if hi * step > cap:
        hi = cap // step + 1
        if fits((hi - 1) * step):
            return (hi - 1) * step
    # fits(lo*step) true, fits(hi*step) false
    while hi - lo > 1:
        mid = (lo + hi) // 2
        if fits(mid * step):
            lo = mid
        else:
            hi = mid
    return lo * step


def max_length(kind, d, h, f, causal, dtype, budget: int, layers: int = 1, step: int = 128,
               cap: int = 1 << 22) -> dict:
    def unchunked(N):
        return profile(block(kind, N, d, h, f, causal, dtype, name="maxlen", layers=layers)).peak_bytes < budget

    def chunked(N):
        return select(block(kind, N, d, h, f, causal, dtype, name="maxlen", layers=layers), budget).feasible

    nu = _largest(unchunked, step, cap)
    nc = _largest(chunked, step, cap)
    return {"unchunked": nu, "chunked": nc, "ratio": (nc / nu) if nu else None}
