"""search (the caller that chooses the microbatch and pack-size knobs) vs the
reference's own search on its test presets: same best configuration, same
estimate, same candidate log (golden: oracle/make_golden_search.py)."""
import pytest

import paper_2202_01306_b200 as H
from conftest import golden
from paper_2202_01306_b200.search import SearchSpec, Strategy, greedy_baseline, search


@pytest.mark.parametrize("case", golden("search.json")["cases"], ids=lambda c: c["name"])
def test_search_matches_reference(case):
    prof = H.synth_profiles(H.SynthSpec(**case["synth"]))
    n, alpha, beta = case["machine"]
    m = H.MachineModel(gpu_count=n, gpu_mem_capacity=alpha, pcie_bandwidth=beta)
    sp = dict(case["spec"])
    if "mode" in sp:
        sp["mode"] = H.Mode(sp["mode"])
    if "strategy" in sp:
        sp["strategy"] = Strategy(sp["strategy"])
    s = SearchSpec(**sp)
    res = search(s, m, prof)
    b = res.best
    assert [b.u_f, [list(p) for p in b.p_f], b.u_b, [list(p) for p in b.p_b]] == case["best"]
    assert res.best_time_ns == case["best_time_ns"]
    assert res.explored == case["explored"]
    assert [[c.u_f, c.u_b, c.pf_count, c.pb_count, c.time_ns, c.note] for c in res.log] == case["log"]
    g, gt = greedy_baseline(s, m, prof)
    assert [g.u_f, [list(p) for p in g.p_f], g.u_b, [list(p) for p in g.p_b], gt] == case["greedy"]


def test_infeasible_space_raises():
    prof = H.synth_profiles(H.SynthSpec(layer_count=12, preset="irregular", seed=5, u_max=16,
                                        w_bytes=64 << 20, act_bytes_per_u=24 << 20))
    with pytest.raises(H.NoFeasibleConfigurationError):
        search(SearchSpec(minibatch=4), H.MachineModel(gpu_count=2, gpu_mem_capacity=1 << 20,
                                                       pcie_bandwidth=16 << 30), prof)
