"""Gantt charts of simulated and MEASURED iteration traces (the reference's
`gantt.render_gantt`, `gantt.py:38-126`, for the path's TraceEvents).

Sources are a :class:`SimReport` (``simulate`` estimate, or
``HarmonyRuntime.report()`` / ``execute`` whose events are CUDA-event
timestamps) or a plain sequence of :class:`TraceEvent`.  Output is
deterministic for identical input.

* ``render_gantt(src, "text")`` -- one row per resource, time bucketed into
  ``width`` columns; a column shows the event kind covering most of it
  (F / B / U compute, W / K / x / y swaps, ``=`` peer copies).
* ``render_gantt(src, "svg")`` -- a standalone SVG, one rectangle per event.
* ``render_comparison(estimated, measured)`` -- both traces on one time axis
  (SVG), the estimator-vs-real view of SURVEY §8f row 2 (`PAPER.md:776`).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Sequence
from xml.sax.saxutils import escape

from .simulator import SimReport, TraceEvent


@dataclass(frozen=True)
class GanttAnnotation:
    resource: str
    start_ns: int
    end_ns: int
    label: str


# one glyph / colour per event kind
_GLYPH = {"W": "W", "K": "K", "dW": "d", "X": "x", "Y": "y", "dX": "x", "dY": "y", "sX": "s"}
_COLOUR = {"F": "#4c78a8", "B": "#f58518", "U": "#54a24b", "W": "#b279a2", "K": "#9d755d", "sX": "#bab0ac",
           "X": "#72b7b2", "Y": "#72b7b2", "dX": "#e45756", "dY": "#e45756", "dW": "#eeca3b"}


def _events(src) -> list[TraceEvent]:
    ev = list(src.trace) if isinstance(src, SimReport) else list(src)
    return sorted(ev, key=lambda e: (e.resource, e.start_ns, e.end_ns, e.task, e.label))


def _key(e: TraceEvent) -> str:
    """Compute events are keyed by their task type (label starts F / B / U)."""
    if e.kind == "compute":
        return e.label[:1] if e.label[:1] in ("F", "B", "U") else "F"
    return e.kind


def _glyph(e: TraceEvent) -> str:
    k = _key(e)
    if "p2p" in e.label:
        return "="
    return k if k in ("F", "B", "U") else _GLYPH.get(k, "#")


def _resource_order(events: Sequence[TraceEvent]) -> list[str]:
    """gpuN lanes in device order (compute, swap_in, swap_out, p2p ...), then host lanes."""
    def rank(r: str):
        dev, _, lane = r.partition(".")
        num = int("".join(ch for ch in dev if ch.isdigit()) or 0)
        return (0 if dev.startswith("gpu") else 1, num, lane)
    return sorted({e.resource for e in events}, key=rank)


def render_gantt(source, fmt: str = "text", annotations: Sequence[GanttAnnotation] = (), width: int = 100,
                 title: str = "") -> str:
    if fmt == "text":
        return _text(_events(source), annotations, width)
    if fmt == "svg":
        return _svg([(title, _events(source))], annotations)
    raise ValueError(f"unknown format {fmt!r}")


def render_comparison(estimated, measured, title: str = "") -> str:
    """Estimated and measured traces stacked on one time axis (SVG)."""
    return _svg([(f"{title} estimated".strip(), _events(estimated)), (f"{title} measured".strip(), _events(measured))],
                ())


def _text(events: list[TraceEvent], annotations: Sequence[GanttAnnotation], width: int) -> str:
    if not events:
        return "gantt (empty)\n"
    t0 = min(e.start_ns for e in events)
    span = max(e.end_ns for e in events) - t0
    col_ns = max(1, -(-span // width))
    lanes = _resource_order(events)
    label_w = max(len(r) for r in lanes)
    out = [f"gantt span={span} ns, {col_ns} ns per column"]
    for lane in lanes:
        cover = [dict() for _ in range(width)]  # column -> glyph -> covered ns
        for e in events:
            if e.resource != lane or e.end_ns <= e.start_ns:
                continue
            a, b = e.start_ns - t0, e.end_ns - t0
            for c in range(a // col_ns, min(width - 1, (b - 1) // col_ns) + 1):
                lo, hi = max(a, c * col_ns), min(b, (c + 1) * col_ns)
                if hi > lo:
                    g = _glyph(e)
                    cover[c][g] = cover[c].get(g, 0) + hi - lo
        row = "".join(max(sorted(c.items()), key=lambda kv: kv[1])[0] if c else "." for c in cover)
        busy = sum(e.end_ns - e.start_ns for e in events if e.resource == lane)
        out.append(f"{lane:<{label_w}} |{row}| {100.0 * busy / span:5.1f}%")
    for an in annotations:
        out.append(f"  note {an.resource} [{an.start_ns - t0}, {an.end_ns - t0}) ns: {an.label}")
    out.append("legend: F/B/U compute, W/K weight/optimizer swaps, s stash, x/y activations, = peer copy, . idle")
    return "\n".join(out) + "\n"


def _svg(panels: list[tuple[str, list[TraceEvent]]], annotations: Sequence[GanttAnnotation]) -> str:
    lane_h, left, chart_w, head = 22, 170, 1100, 28
    allev = [e for _, ev in panels for e in ev]
    t0 = min((e.start_ns for e in allev), default=0)
    span = max(1, max((e.end_ns for e in allev), default=1) - t0)
    x = lambda t: left + chart_w * (t - t0) / span  # noqa: E731
    parts, y = [], 0
    for title, ev in panels:
        lanes = _resource_order(ev)
        parts.append(f'<text x="4" y="{y + 18}" font-weight="bold">{escape(title or "trace")}</text>')
        y += head
        for i, lane in enumerate(lanes):
            ly = y + i * lane_h
            parts.append(f'<text x="4" y="{ly + 15}">{escape(lane)}</text>')
            parts.append(f'<rect x="{left}" y="{ly}" width="{chart_w}" height="{lane_h - 2}" fill="#f4f4f4"/>')
            for e in ev:
                if e.resource != lane:
                    continue
                w = max(0.5, x(e.end_ns) - x(e.start_ns))
                col = "#17becf" if "p2p" in e.label else _COLOUR.get(_key(e), "#888888")
                parts.append(f'<rect x="{x(e.start_ns):.2f}" y="{ly + 1}" width="{w:.2f}" height="{lane_h - 4}" '
                             f'fill="{col}"><title>{escape(f"task {e.task}: {e.label} [{e.start_ns}, {e.end_ns}) ns")}'
                             f'</title></rect>')
            for an in annotations:
                if an.resource == lane:
                    parts.append(f'<rect x="{x(an.start_ns):.2f}" y="{ly}" width="{max(0.5, x(an.end_ns) - x(an.start_ns)):.2f}" '
                                 f'height="{lane_h - 2}" fill="none" stroke="#d62728" stroke-dasharray="3,2">'
                                 f'<title>{escape(an.label)}</title></rect>')
        y += len(lanes) * lane_h + 8
    # time axis: 10 ticks
    for k in range(11):
        t = t0 + span * k // 10
        parts.append(f'<line x1="{x(t):.2f}" y1="0" x2="{x(t):.2f}" y2="{y}" stroke="#cccccc" stroke-width="0.5"/>')
        parts.append(f'<text x="{x(t):.2f}" y="{y + 14}" font-size="10" text-anchor="middle">{(t - t0) / 1e6:.2f} ms</text>')
    h = y + 24
    return (f'<svg xmlns="http://www.w3.org/2000/svg" width="{left + chart_w + 20}" height="{h}" '
            f'font-family="monospace" font-size="12">\n' + "\n".join(parts) + "\n</svg>\n")
