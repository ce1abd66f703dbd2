"""Wire formats: documents written by the reference load here and re-emit
identically; our estimate of the reference's task graph reproduces its
sim_report document exactly."""
import paper_2202_01306_b200 as H
from conftest import golden
from paper_2202_01306_b200 import fileio as F


def test_reference_documents_round_trip():
    docs = golden("fileio.json")
    m = F.machine_from_doc(docs["machine"])
    assert F.machine_to_doc(m) == docs["machine"]
    p = F.profileset_from_doc(docs["profile_set"])
    assert F.profileset_to_doc(p) == docs["profile_set"]
    c = F.config_from_doc(docs["configuration"])
    assert F.config_to_doc(c) == docs["configuration"]
    g = F.taskgraph_from_doc(docs["task_graph"])
    assert F.taskgraph_to_doc(g) == docs["task_graph"]
    s = F.samples_from_doc(docs["profile_samples"])
    assert F.samples_to_doc(s, seed=7) == docs["profile_samples"]
    rep = F.report_from_doc(docs["sim_report"])
    assert F.report_to_doc(rep) == docs["sim_report"]
    # our estimator on the reference's own graph reproduces its report document
    ours = H.simulate(g, m, p)
    assert F.report_to_doc(ours) == docs["sim_report"]
    assert F.trace_to_csv(ours) == docs["trace_csv"]


def test_measured_report_carries_ledger(tmp_path):
    docs = golden("fileio.json")
    g = F.taskgraph_from_doc(docs["task_graph"])
    rep = H.simulate(g, F.machine_from_doc(docs["machine"]), F.profileset_from_doc(docs["profile_set"]))
    rep.measured = True
    path = tmp_path / "r.json"
    F.save_json(F.report_to_doc(rep), path)
    back = F.report_from_doc(F.load_json(path))
    assert back.measured and back.ledger == rep.ledger


def test_cli_simulate_and_search(tmp_path):
    """CLI on the reference's documents; exit codes as the reference's CLI."""
    import json
    from paper_2202_01306_b200.cli import main
    docs = golden("fileio.json")
    for name in ("machine", "profile_set", "configuration"):
        (tmp_path / f"{name}.json").write_text(json.dumps(docs[name]))
    rc = main(["simulate", "--machine", str(tmp_path / "machine.json"), "--profiles",
               str(tmp_path / "profile_set.json"), "--config", str(tmp_path / "configuration.json"),
               "--out", str(tmp_path / "r.json")])
    assert rc == 0
    assert F.load_json(tmp_path / "r.json") == docs["sim_report"]
    (tmp_path / "spec.json").write_text(json.dumps({"format_version": 1, "kind": "search_spec",
                                                    "minibatch": 6, "mode": "pp"}))
    assert main(["search", "--machine", str(tmp_path / "machine.json"), "--profiles",
                 str(tmp_path / "profile_set.json"), "--spec", str(tmp_path / "spec.json"),
                 "--out-dir", str(tmp_path / "run")]) == 0
    bad = dict(docs["configuration"], u_f=99)
    (tmp_path / "bad.json").write_text(json.dumps(bad))
    assert main(["simulate", "--machine", str(tmp_path / "machine.json"), "--profiles",
                 str(tmp_path / "profile_set.json"), "--config", str(tmp_path / "bad.json"),
                 "--out", str(tmp_path / "x.json")]) == 2
