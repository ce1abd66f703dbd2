"""bench.py's phase-serialised link bound on the headline plan (CPU): the
forward window moves 6.55 GB in / 0.42 GB out, the backward + update window
20.1 GB in / 19.7 GB out, and the bound equals the sum of each
window's own max over directions."""
import os
import sys

import pytest

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def test_phase_bound_headline_plan():
    import bench
    import paper_2202_01306_b200 as H
    from paper_2202_01306_b200.model import GPT_PRESETS, gpt_machine, gpt_profiles
    spec = GPT_PRESETS["gpt2-xl"]
    packs = tuple((i, min(i + 8, spec.n_layer) - 1) for i in range(0, spec.n_layer, 8))
    m = gpt_machine(1, alpha_bytes=32 << 30)
    prof = gpt_profiles(spec)
    g = H.generate_task_graph(H.Configuration(4, packs, 4, packs, 16, H.Mode.DP), m, prof)
    sim = H.simulate(g, m, prof)
    pcie = {"h2d": 55.58, "d2h": 56.08, "bidir": 90.65}
    t = bench.phase_bound_s(g, sim.ledger, pcie)
    fwd_in, fwd_out, bwd_in, bwd_out = 6.5526912e9, 0.419495936e9, 20.077569536e9, 19.6580736e9
    want = max(fwd_in / 55.58e9, fwd_out / 56.08e9, (fwd_in + fwd_out) / 90.65e9) + \
        max(bwd_in / 55.58e9, bwd_out / 56.08e9, (bwd_in + bwd_out) / 90.65e9)
    assert t == pytest.approx(want, rel=1e-9)
    # the whole-step bound is never above the phase-serialised one
    tot_in, tot_out = fwd_in + bwd_in, fwd_out + bwd_out
    assert max(tot_in / 55.58e9, tot_out / 56.08e9, (tot_in + tot_out) / 90.65e9) <= t
