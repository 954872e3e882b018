"""Gate bookkeeping for the GPU parity tests: every gate records observed / tolerance before it
asserts, so the margins are visible (a 100x regression that stays inside a loose tolerance shows up
in the summary) and the branches taken by the outcome logic (T7) are counted.

pytest prints the summary at the end of the session (tests/conftest.py) and writes it to
``gpurun_out/gate_margins.json`` when that directory exists.
"""
from __future__ import annotations

import math
from collections import defaultdict

RECORDS: dict[str, list[tuple[str, float, float]]] = defaultdict(list)
BRANCHES: dict[str, int] = defaultdict(int)


def gate(name: str, observed: float, tol: float, case: str = "") -> float:
    """Record and assert observed <= tol; returns the margin observed / tol."""
    observed, tol = float(observed), float(tol)
    ratio = observed / tol if tol > 0 else (0.0 if observed == 0 else math.inf)
    RECORDS[name].append((case, observed, tol))
    assert observed <= tol, f"gate {name} [{case}]: observed {observed:.3e} > tolerance {tol:.3e}"
    return ratio


def note(name: str, observed: float, tol: float, case: str = "") -> float:
    """Record a margin without asserting (report-only comparisons)."""
    observed, tol = float(observed), float(tol)
    RECORDS[name].append((case, observed, tol))
    return observed / tol if tol > 0 else math.inf


def branch(name: str) -> None:
    BRANCHES[name] += 1


def summary() -> dict:
    out = {}
    for name, rows in sorted(RECORDS.items()):
        ratios = sorted(o / t if t > 0 else (0.0 if o == 0 else math.inf) for _, o, t in rows)
        worst = max(rows, key=lambda r: r[1] / r[2] if r[2] > 0 else math.inf)
        out[name] = dict(n=len(rows), max_ratio=ratios[-1], median_ratio=ratios[len(ratios) // 2],
                         worst_case=worst[0], worst_observed=worst[1], worst_tol=worst[2])
    records = {name: [[case, o, t] for case, o, t in rows] for name, rows in sorted(RECORDS.items())}
    return dict(gates=out, branches=dict(sorted(BRANCHES.items())), records=records)
