"""Trace CSV artifacts (evaluation.py:154-200 of the reference): lossless
17-significant-digit rows ``problem, solver, stage, iteration, cost,
elapsed_seconds``.  The performance-profile machinery (evaluation.py:62-147) is
post-processing outside the hot path and is not part of this package."""

from __future__ import annotations

import csv
from pathlib import Path
from typing import IO, Iterable

from .types import ConvergenceTrace, TraceRecord

TRACE_HEADER = ["problem", "solver", "stage", "iteration", "cost", "elapsed_seconds"]


def _fmt(x: float) -> str:
    return format(x, ".17g")


def _open_sink(sink, mode: str):
    if isinstance(sink, (str, Path)):
        return open(sink, mode, newline=""), True
    return sink, False


def write_trace_csv(traces: Iterable[ConvergenceTrace], sink: str | Path | IO[str]) -> None:
    fh, owned = _open_sink(sink, "w")
    try:
        w = csv.writer(fh)
        w.writerow(TRACE_HEADER)
        for t in traces:
            for rec in t.records:
                w.writerow([t.problem_id, t.solver_id, t.stage, rec.iteration,
                            _fmt(rec.cost), _fmt(rec.elapsed_seconds)])
    finally:
        if owned:
            fh.close()


def read_trace_csv(source: str | Path | IO[str]) -> list[ConvergenceTrace]:
    fh, owned = _open_sink(source, "r")
    try:
        rd = csv.reader(fh)
        header = next(rd, None)
        if header != TRACE_HEADER:
            raise ValueError(f"unexpected trace CSV header: {header}")
        grouped: dict[tuple[str, str, str], list[TraceRecord]] = {}
        for row in rd:
            if not row:
                continue
            problem, solver, stage, it, cost, elapsed = row
            grouped.setdefault((problem, solver, stage), []).append(
                TraceRecord(int(it), float(cost), float(elapsed)))
        return [ConvergenceTrace(solver, problem, stage, recs, recs[0].cost)
                for (problem, solver, stage), recs in grouped.items()]
    finally:
        if owned:
            fh.close()
