"""Work model of basic (l = 2) HouseHT -- measurement logic only (no method arithmetic).

F_model(n, nb) is SURVEY.md Appendix A's flop count of Algorithm 1
with Q and Z accumulated and no iterative refinement: panel solves/residuals/A*v
(sec. 3.2), the Remark-2 GEMM and the absorption 72 n k m + 18 k m^2 per
panel (sec. 3.3).  The roofline model splits the work into the level-3
flops of the absorption (FP64 tensor pipe) and the level-2 HBM bytes of the panel.
"""
from __future__ import annotations


def model_flops(n: int, nb: int) -> float:
    """F_model (App. A): fixed per (n, nb), the common denominator of both bench arms."""
    tot = 0.0
    s0 = 0
    while s0 <= n - 3:
        k = min(nb, n - 2 - s0)
        p0 = s0 + 1
        M = n - p0
        J = s0 + k
        m = n - J - 1
        for i in range(k):
            tot += M * M + (M * M if i > 0 else 0.0) + 2.0 * M * (n - s0 - i - 1)
        tot += 2.0 * p0 * M * k + 4.0 * p0 * k * k
        tot += 72.0 * n * k * m + 18.0 * k * m * m
        s0 = J
    return tot


def roofline_seconds(flops_level3: float, panel_bytes: float, p64_tflops: float, hbm_gbs: float) -> float:
    """T_roof = F_L3 / P64 + B_L2 / BW: the absorption's level-3 flops at the
    FP64 tensor peak plus the panel's level-2 bytes at the HBM peak (no overlap assumed)."""
    return flops_level3 / (p64_tflops * 1e12) + panel_bytes / (hbm_gbs * 1e9)
