"""ORACLE (test infrastructure only -- never imported by the product path).

torch-CPU fp32 restatement of one Harmony training iteration for the GPT
layer chain (SURVEY §8c "Numerics"):
synchronous SGD with the single-device loss (mean token cross-entropy over
the minibatch), gradients accumulated over the microbatch members of each
backward group, then a jit Adam update per pack.  Because every backward
task reads its pack's weights before that pack's update and consumes
gradients computed with pre-update weights, the iteration equals full-batch
backprop followed by Adam on every pack -- which is what this module computes,
member by member in the schedule's F/B order.

Parity is UNPINNED by the reference (it has no tensor arithmetic); this
restatement is checked by tests/test_gpt_oracle.py against torch.autograd on
a straightforward nn-style model and against torch.optim.Adam.

The parameter layout mirrors GPTSpec.layer_segments (flat fp32 per layer).
"""

from __future__ import annotations

import math

import numpy as np
import torch
import torch.nn.functional as F


def _segments(spec, L):
    return spec.layer_segments(L)


class GPTOracle:
    def __init__(self, spec, w_flat: np.ndarray, w_off: np.ndarray, lr=1e-4, betas=(0.9, 0.999), eps=1e-8):
        self.spec = spec
        self.w = torch.tensor(np.array(w_flat, dtype=np.float32, copy=True))
        self.m = torch.zeros_like(self.w)
        self.v = torch.zeros_like(self.w)
        self.off = [int(x) for x in w_off]
        self.lr, self.b1, self.b2, self.eps = lr, betas[0], betas[1], eps
        self.t = 0

    def _views(self, flat, L):
        out, o = {}, self.off[L]
        d, vp = self.spec.d_model, self.spec.vocab_padded
        shapes = {"wte": (vp, d), "wpe": (self.spec.seq_len, d), "w_qkv": (3 * d, d), "w_proj": (d, d),
                  "w_fc1": (4 * d, d), "w_fc2": (d, 4 * d), "w_head": (vp, d)}
        for name, n in _segments(self.spec, L):
            t = flat[o:o + n]
            out[name] = t.view(*shapes[name]) if name in shapes else t
            o += n
        return out

    def _block(self, p, x):
        s = self.spec
        B, S, d = x.shape
        H, Dh = s.n_head, s.head_dim
        h = F.layer_norm(x, (d,), p["ln1_g"], p["ln1_b"], 1e-5)
        qkv = h @ p["w_qkv"].t() + p["b_qkv"]
        q, k, v = qkv.view(B, S, 3, H, Dh).permute(2, 0, 3, 1, 4)
        att = (q @ k.transpose(-1, -2)) / math.sqrt(Dh)
        if s.causal:
            att = att.masked_fill(torch.triu(torch.ones(S, S, dtype=torch.bool), 1), float("-inf"))
        o = (torch.softmax(att, -1) @ v).permute(0, 2, 1, 3).reshape(B, S, d)
        x = x + o @ p["w_proj"].t() + p["b_proj"]
        h = F.layer_norm(x, (d,), p["ln2_g"], p["ln2_b"], 1e-5)
        a = F.gelu(h @ p["w_fc1"].t() + p["b_fc1"], approximate="tanh")
        return x + a @ p["w_fc2"].t() + p["b_fc2"]

    def loss_sum(self, flat, tokens, labels):
        """Summed token CE of one member (tokens/labels int64 [u, S]).
        ``flat`` is the flat parameter vector or per-layer view dicts."""
        s = self.spec
        x = None
        for L in range(s.n_layer):
            p = flat[L] if isinstance(flat, list) else self._views(flat, L)
            if L == 0:
                x = p["wte"][tokens] + p["wpe"][None, :, :]
            x = self._block(p, x)
            if L == s.n_layer - 1:
                h = F.layer_norm(x, (s.d_model,), p["lnf_g"], p["lnf_b"], 1e-5)
                logits = h @ p["w_head"][: s.vocab].t()
                return F.cross_entropy(logits.reshape(-1, s.vocab), labels.reshape(-1), reduction="sum")
        raise AssertionError

    def step(self, tokens: np.ndarray, labels: np.ndarray, groups) -> float:
        """One iteration over the minibatch split into ``groups`` members."""
        tokens = torch.as_tensor(tokens, dtype=torch.long)
        labels = torch.as_tensor(labels, dtype=torch.long)
        n_tok = tokens.numel()
        # one autograd leaf per parameter segment (views of a copy of W): the
        # backward of a slice of one flat leaf would materialise a zero tensor
        # of the WHOLE model per segment (minutes per iteration at 1.5 B)
        base = self.w.clone()
        leaves = []
        for L in range(self.spec.n_layer):
            leaves.append({k: t.requires_grad_(True) for k, t in self._views(base, L).items()})
        total = 0.0
        s0 = 0
        for u in groups:
            ls = self.loss_sum(leaves, tokens[s0:s0 + u], labels[s0:s0 + u])
            (ls / n_tok).backward()
            total += ls.item()
            s0 += u
        g = torch.zeros_like(self.w)
        for L in range(self.spec.n_layer):
            o = self.off[L]
            for name, n in _segments(self.spec, L):
                t = leaves[L][name]
                if t.grad is not None:
                    g[o:o + n] = t.grad.reshape(-1)
                o += n
        del leaves, base
        self.t += 1
        # torch.optim.Adam (no weight decay), elementwise over every pack
        self.m.lerp_(g, 1 - self.b1)
        self.v.mul_(self.b2).addcmul_(g, g, value=1 - self.b2)
        bc1 = 1 - self.b1 ** self.t
        bc2 = 1 - self.b2 ** self.t
        denom = (self.v.sqrt() / math.sqrt(bc2)).add_(self.eps)
        self.w.addcdiv_(self.m, denom, value=-self.lr / bc1)
        return total / n_tok
