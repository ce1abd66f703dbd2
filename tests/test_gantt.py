"""Gantt rendering of simulated / measured traces (gantt.py; the reference's
`gantt.py:38-126` behaviour: one lane per resource, deterministic output)."""

import xml.etree.ElementTree as ET

import paper_2202_01306_b200 as H
from paper_2202_01306_b200 import cli
from paper_2202_01306_b200 import fileio as F
from paper_2202_01306_b200.gantt import GanttAnnotation, render_comparison, render_gantt
from paper_2202_01306_b200.model import GPT_PRESETS, gpt_profiles


def _report(n=2, mode=H.Mode.PP):
    spec = GPT_PRESETS["tiny"]
    prof = gpt_profiles(spec)
    m = H.MachineModel(gpu_count=n, gpu_mem_capacity=4 << 30, pcie_bandwidth=55_000_000_000)
    packs = ((0, 1), (2, 3))
    g = H.generate_task_graph(H.Configuration(4, packs, 4, packs, 16, mode), m, prof)
    return H.simulate(g, m, prof)


def test_text_lanes_and_determinism():
    r = _report()
    a = render_gantt(r, width=80)
    assert a == render_gantt(r, width=80)
    lines = a.splitlines()
    lanes = {e.resource for e in r.trace}
    body = [ln for ln in lines[1:] if "|" in ln]
    assert len(body) == len(lanes)
    # gpu lanes first, in device order
    assert body[0].startswith("gpu0.") and body[-1].startswith("cpu")
    for ln in body:
        assert len(ln.split("|")[1]) == 80
    assert "F" in a and "B" in a and "U" in a and "W" in a and "K" in a


def test_empty_and_unknown_format():
    assert render_gantt([], "text").startswith("gantt")
    try:
        render_gantt(_report(), "png")
    except ValueError:
        pass
    else:
        raise AssertionError("unknown format accepted")


def test_svg_parses_and_has_one_rect_per_event():
    r = _report()
    ann = [GanttAnnotation("gpu0.compute", 0, 1000, "note")]
    svg = render_gantt(r, "svg", annotations=ann)
    root = ET.fromstring(svg)
    rects = [e for e in root.iter() if e.tag.endswith("rect")]
    lanes = {e.resource for e in r.trace}
    # lane backgrounds + events + the annotation
    assert len(rects) == len(lanes) + len(r.trace) + 1
    cmp = render_comparison(r, r, title="tiny")
    root = ET.fromstring(cmp)
    texts = [e.text for e in root.iter() if e.tag.endswith("text")]
    assert "tiny estimated" in texts and "tiny measured" in texts


def test_cli_gantt_roundtrip(tmp_path, capsys):
    r = _report(1)
    p = tmp_path / "r.json"
    F.save_json(F.report_to_doc(r), p)
    assert cli.main(["gantt", "--report", str(p), "--width", "60"]) == 0
    out = capsys.readouterr().out
    assert out == render_gantt(F.report_from_doc(F.load_json(p)), width=60)
    svg = tmp_path / "g.svg"
    assert cli.main(["gantt", "--report", str(p), "--compare", str(p), "--fmt", "svg", "--out", str(svg)]) == 0
    ET.parse(svg)
    assert cli.main(["gantt", "--report", str(p), "--compare", str(p), "--fmt", "text"]) == 2
