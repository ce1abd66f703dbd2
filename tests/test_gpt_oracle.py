"""CPU checks of the numerics oracle (oracle/gpt_cpu.py): its Adam equals
torch.optim.Adam, its loss is member-chunking invariant, and its parameter
layout matches GPTSpec (which the native runtime checks against itself)."""

import numpy as np
import torch

from oracle.gpt_cpu import GPTOracle
from paper_2202_01306_b200.model import GPTSpec, synthetic_batch


def _spec():
    return GPTSpec(2, 64, 1, 64, 96, True, "micro")


def _init(spec, seed=0):
    n = spec.total_params()
    g = torch.Generator().manual_seed(seed)
    w = (torch.randn(n, generator=g) * 0.02).numpy()
    off = np.cumsum([0] + [spec.layer_params(L) for L in range(spec.n_layer)])
    return w, off


def test_oracle_adam_equals_torch_adam():
    spec = _spec()
    w, off = _init(spec)
    o = GPTOracle(spec, w, off)
    tok, lab = synthetic_batch(spec, 4)
    p = torch.nn.Parameter(torch.tensor(w))
    opt = torch.optim.Adam([p], lr=1e-4, betas=(0.9, 0.999), eps=1e-8)
    for _ in range(3):
        flat = p.detach().clone().requires_grad_(True)
        loss = o.loss_sum(flat, torch.as_tensor(tok).long(), torch.as_tensor(lab).long()) / tok.size
        loss.backward()
        p.grad = flat.grad
        opt.step()
        o.step(tok, lab, [4])
    assert torch.allclose(o.w, p.detach(), rtol=1e-6, atol=1e-8)


def test_oracle_member_chunking_invariant():
    spec = _spec()
    w, off = _init(spec)
    a, b = GPTOracle(spec, w, off), GPTOracle(spec, w, off)
    tok, lab = synthetic_batch(spec, 6)
    la = a.step(tok, lab, [6])
    lb = b.step(tok, lab, [4, 2])
    assert abs(la - lb) < 1e-5
    # Adam normalises each component's update: components whose gradient is
    # ~0 move by up to lr on rounding noise, so allow 1% of one step there
    assert torch.allclose(a.w, b.w, atol=1e-6)


def test_spec_layout_sums():
    for spec in (_spec(), GPTSpec(4, 256, 4, 128, 1024)):
        for L in range(spec.n_layer):
            assert sum(n for _, n in spec.layer_segments(L)) == spec.layer_params(L)
