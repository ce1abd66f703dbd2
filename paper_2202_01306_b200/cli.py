"""Command line for the path (the reference's `simulate` / `search` plus the
new `execute`), reading and writing the reference's JSON documents.

    python -m paper_2202_01306_b200 simulate --machine m.json --profiles p.json --config c.json --out r.json
    python -m paper_2202_01306_b200 search   --machine m.json --profiles p.json --spec s.json --out-dir run/
    python -m paper_2202_01306_b200 execute  --preset gpt2-xl --machine m.json --config c.json --steps 3 --out r.json
    python -m paper_2202_01306_b200 profile  --preset gpt2-xl --out p.json
    python -m paper_2202_01306_b200 gantt    --report measured.json [--compare estimate.json] --fmt svg --out g.svg

Exit codes follow the reference (`cli.py:66-71`): 0 ok, 2 validation error,
3 infeasible, 4 internal / device error.
"""

from __future__ import annotations

import argparse
import os
import sys

from . import fileio as F
from .errors import (LayerTooLargeError, NoFeasibleConfigurationError, UnpackableError, ValidationError,
                     WrapschedError)


def _simulate(a) -> int:
    from .simulator import simulate
    from .taskgraph import generate_task_graph
    m = F.machine_from_doc(F.load_json(a.machine))
    p = F.profileset_from_doc(F.load_json(a.profiles))
    g = generate_task_graph(F.config_from_doc(F.load_json(a.config)), m, p)
    rep = simulate(g, m, p, check_memory=a.check_memory)
    F.save_json(F.report_to_doc(rep), a.out)
    if a.trace_csv:
        open(a.trace_csv, "w").write(F.trace_to_csv(rep))
    print(f"makespan {rep.makespan_ns / 1e6:.3f} ms, swap {sum(rep.per_gpu_swap_bytes.values()) / 1e9:.3f} GB")
    return 0


def _search(a) -> int:
    from .search import search
    m = F.machine_from_doc(F.load_json(a.machine))
    p = F.profileset_from_doc(F.load_json(a.profiles))
    res = search(F.search_spec_from_doc(F.load_json(a.spec)), m, p)
    os.makedirs(a.out_dir, exist_ok=True)
    F.save_json(F.search_result_to_doc(res), os.path.join(a.out_dir, "search_result.json"))
    F.save_json(F.config_to_doc(res.best), os.path.join(a.out_dir, "best_config.json"))
    print(f"best {res.best_time_ns / 1e6:.3f} ms over {res.explored} candidates in {res.wall_time_s:.2f} s")
    return 0


def _execute(a) -> int:
    from .model import GPT_PRESETS, gpt_profiles, synthetic_batch
    from .runtime import execute
    from .taskgraph import generate_task_graph
    spec = GPT_PRESETS[a.preset]
    m = F.machine_from_doc(F.load_json(a.machine))
    p = F.profileset_from_doc(F.load_json(a.profiles)) if a.profiles else gpt_profiles(spec)
    cfg = F.config_from_doc(F.load_json(a.config))
    g = generate_task_graph(cfg, m, p)
    rep = execute(g, m, p, model=spec, batch=synthetic_batch(spec, cfg.minibatch), steps=a.steps)
    F.save_json(F.report_to_doc(rep), a.out)
    if a.gantt:  # estimate and measurement of the same graph on one time axis
        from .gantt import render_comparison
        from .simulator import simulate
        open(a.gantt, "w").write(render_comparison(simulate(g, m, p), rep, title=a.preset))
    print(f"measured iteration {rep.makespan_ns / 1e6:.3f} ms; {rep.caveats[-1]}")
    return 0


def _gantt(a) -> int:
    from .gantt import render_comparison, render_gantt
    rep = F.report_from_doc(F.load_json(a.report))
    if a.compare:
        if a.fmt != "svg":
            raise ValidationError("--compare renders SVG only")
        doc = render_comparison(F.report_from_doc(F.load_json(a.compare)), rep)
    else:
        doc = render_gantt(rep, a.fmt, width=a.width)
    if a.out:
        open(a.out, "w").write(doc)
    else:
        sys.stdout.write(doc)
    return 0


def _profile(a) -> int:
    from .model import GPT_PRESETS
    from .profiling import profile_gpt
    prof, samples = profile_gpt(GPT_PRESETS[a.preset], u_values=tuple(a.u))
    F.save_json(F.profileset_to_doc(prof), a.out)
    if a.samples:
        F.save_json(F.samples_to_doc(samples), a.samples)
    return 0


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="paper_2202_01306_b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    s = sub.add_parser("simulate")
    s.add_argument("--machine", required=True)
    s.add_argument("--profiles", required=True)
    s.add_argument("--config", required=True)
    s.add_argument("--out", required=True)
    s.add_argument("--trace-csv")
    s.add_argument("--check-memory", action="store_true")
    s.set_defaults(fn=_simulate)
    s = sub.add_parser("search")
    s.add_argument("--machine", required=True)
    s.add_argument("--profiles", required=True)
    s.add_argument("--spec", required=True)
    s.add_argument("--out-dir", required=True)
    s.set_defaults(fn=_search)
    s = sub.add_parser("execute")
    s.add_argument("--preset", required=True)
    s.add_argument("--machine", required=True)
    s.add_argument("--config", required=True)
    s.add_argument("--profiles")
    s.add_argument("--steps", type=int, default=1)
    s.add_argument("--out", required=True)
    s.add_argument("--gantt", help="SVG of the estimated and the measured trace")
    s.set_defaults(fn=_execute)
    s = sub.add_parser("gantt")
    s.add_argument("--report", required=True, help="sim_report JSON (simulate or execute)")
    s.add_argument("--compare", help="a second report drawn above it (e.g. the estimate)")
    s.add_argument("--fmt", choices=("text", "svg"), default="text")
    s.add_argument("--width", type=int, default=100)
    s.add_argument("--out")
    s.set_defaults(fn=_gantt)
    s = sub.add_parser("profile")
    s.add_argument("--preset", required=True)
    s.add_argument("--u", type=int, nargs="+", default=[1, 2, 4])
    s.add_argument("--out", required=True)
    s.add_argument("--samples")
    s.set_defaults(fn=_profile)
    return ap


def main(argv=None) -> int:
    a = build_parser().parse_args(argv)
    try:
        return a.fn(a)
    except (NoFeasibleConfigurationError, LayerTooLargeError, UnpackableError) as exc:
        print(f"infeasible: {exc}", file=sys.stderr)
        return 3
    except ValidationError as exc:
        print(f"validation error: {exc}", file=sys.stderr)
        return 2
    except WrapschedError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 4


if __name__ == "__main__":
    sys.exit(main())
