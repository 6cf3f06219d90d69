"""Closed-form budget models (host logic, no device code).

memory_budget  -- Table 1a 'Compression ratio of GPU' (§3.3)
comm_overhead  -- §3.3 'Communication overhead': retain·n·L·H·bytes
cost_per_query -- Table 1b / §3.2 P:229 per decode query
algorithmic_bytes -- DESIGN.md §6: the bytes the method itself must move per
                     (batch, layer, KV head) per decode step; the roofline numerator.
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class BudgetReport:
    K: float
    V: float
    total: float


def memory_budget(d: int, g: int | None, value_offloaded: bool) -> BudgetReport:
    """Table 1a: K fraction = g/d with 2-byte indices vs 2-byte elements;
    V fraction 0 when offloaded; total = mean of the two."""
    if g is not None and (g <= 0 or d % g):
        raise ValueError("g must divide d")
    k = 100.0 if g is None else 100.0 * g / d
    v = 0.0 if value_offloaded else 100.0
    return BudgetReport(k, v, (k + v) / 2.0)


def comm_overhead(n: int, L: int, H: int, retain_fraction: float, bytes_per_score: int) -> float:
    """§3.3: (1/5)·n·L·H·2 Bytes ≈ 102.4 MB at n=1e6, L=32, H=8."""
    if not 0.0 <= retain_fraction <= 1.0:
        raise ValueError("retain_fraction outside [0,1]")
    return retain_fraction * n * L * H * bytes_per_score


def cost_per_query(n: int, d: int, c: int, g: int) -> dict:
    """Per decode query: exact n·d mults; HCAttention d·c mults (T = q̄·C) and
    n·g adds (Eq. 3)."""
    return dict(exact_mults=n * d, approx_mults=d * c, approx_adds=n * g)


def algorithmic_bytes(n: int, g: int, G: int, d: int, c: int, dbar: int, k_sel_total: int,
                      units_sharing_codebook: int) -> dict:
    """Bytes per (batch, layer, KV-head) unit per decode step:
    P codes 2·n·g; selected V rows k_sel_total·d·2 (summed over the G heads);
    codebook share c·dbar·4·g/units; q in + out G·d·(2+4)."""
    return dict(
        P=2 * n * g,
        V=k_sel_total * d * 2,
        C=(g * c * dbar * 4) // max(units_sharing_codebook, 1),
        qo=G * d * (2 + 4),
    )
