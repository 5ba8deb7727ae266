"""Shared helpers for the parity tests (test infrastructure)."""
import numpy as np

from oracle import RefConfig, RefSystem, splitmix_vector, ref_available, OracleSystem, oracle_available


def checker(**kw):
    """The compiled reference when present, else the restatement oracle."""
    if ref_available():
        return RefSystem(RefConfig(**kw))
    return OracleSystem(RefConfig(**kw))


def rel(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    den = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (den if den > 0 else 1.0))


def history_parity(ours: dict, ref: dict, tol=1e-10, iters_slack=1):
    """SURVEY §8c parity rule: iterations +-1, max_k |dr_k|/r_0 <= tol, rel-L2(u) <= tol."""
    assert ours["status"] == ref["status"], (ours["status"], ref["status"])
    assert abs(ours["iterations"] - ref["iterations"]) <= iters_slack, (ours["iterations"], ref["iterations"])
    ra, rb = np.asarray(ours["residual_history"]), np.asarray(ref["residual_history"])
    k = min(len(ra), len(rb))
    r0 = rb[0]
    assert abs(ra[0] - r0) <= 1e-13 * r0
    dr = float(np.max(np.abs(ra[:k] - rb[:k])) / r0)
    assert dr <= tol, dr
    if ours.get("u") is not None:
        assert rel(ours["u"], ref["u"]) <= tol, rel(ours["u"], ref["u"])
    return dr
