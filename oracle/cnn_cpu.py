"""ORACLE (test infrastructure only -- never imported by the product path).

torch-CPU fp32 restatement of one Harmony training iteration for the deep-CNN
layer chain (paper_2202_01306_b200/cnn.py): the same single-device semantics
as oracle/gpt_cpu.py -- mean cross-entropy over
the minibatch, gradients accumulated over the microbatch members, one Adam
step on every pack.  Parity is UNPINNED by the reference (it has no tensor
arithmetic); the layer math is plain torch (conv2d, avg_pool2d, mean, linear)
on the parameters the runtime keeps in its W arena (weights [cout, 3, 3, cin],
permuted here to torch's [cout, cin, 3, 3]).
"""

from __future__ import annotations

import math

import numpy as np
import torch
import torch.nn.functional as F

CONV, DOWN, RES, HEAD, RES2 = 0, 1, 2, 3, 4


class CNNOracle:
    def __init__(self, spec, w_flat: np.ndarray, w_off: np.ndarray, lr=1e-4, betas=(0.9, 0.999), eps=1e-8):
        self.spec = spec
        self.w = torch.tensor(np.array(w_flat, dtype=np.float32, copy=True))
        self.m = torch.zeros_like(self.w)
        self.v = torch.zeros_like(self.w)
        self.off = [int(x) for x in w_off]
        self.lr, self.b1, self.b2, self.eps = lr, betas[0], betas[1], eps
        self.t = 0

    def _raw(self, flat, L):
        out, o = {}, self.off[L]
        for name, shp in self.spec.layer_segments(L):
            n = int(np.prod(shp))
            out[name] = flat[o:o + n].view(*shp)
            o += n
        return out

    def _views(self, flat, L):
        raw = flat[L] if isinstance(flat, list) else self._raw(flat, L)
        return {k: t.permute(0, 3, 1, 2) if t.dim() == 4 else t for k, t in raw.items()}  # [cout, cin, 3, 3]

    def loss_sum(self, flat, images, labels):
        """Summed cross-entropy of one member: images [u, h, w, c] fp32 NHWC."""
        x = images.permute(0, 3, 1, 2)
        outs = []  # every layer's output (res2 adds an earlier one back)
        for L, (t, cin, cout, h, w) in enumerate(self.spec.layers):
            p = self._views(flat, L)
            if t == RES2:
                x = F.relu(F.conv2d(x, p["w1"], p["b1"], padding=1) + outs[self.spec.skips[L]])
                outs.append(x)
                continue
            if t == HEAD:
                pooled = x.mean(dim=(2, 3))
                logits = pooled @ p["w1"][: self.spec.classes].t() + p["b1"][: self.spec.classes]
                return F.cross_entropy(logits, labels, reduction="sum")
            if t == RES:
                hh = F.relu(F.conv2d(x, p["w1"], p["b1"], padding=1))
                x = F.relu(x + F.conv2d(hh, p["w2"], p["b2"], padding=1))
            else:
                x = F.relu(F.conv2d(x, p["w1"], p["b1"], padding=1))
                if t == DOWN:
                    x = F.avg_pool2d(x, 2)
            outs.append(x)
        raise AssertionError("chain without a head")

    def step(self, images, labels, groups) -> float:
        images = torch.as_tensor(images).float()
        labels = torch.as_tensor(labels, dtype=torch.long)
        n = labels.numel()
        # one autograd leaf per parameter segment (a slice of one flat leaf
        # would materialise a whole-model zero tensor per segment in backward)
        base = self.w.clone()
        leaves = [{k: t.requires_grad_(True) for k, t in self._raw(base, L).items()}
                  for L in range(len(self.spec.layers))]
        total, s0 = 0.0, 0
        for u in groups:
            ls = self.loss_sum(leaves, images[s0:s0 + u], labels[s0:s0 + u])
            (ls / n).backward()
            total += ls.item()
            s0 += u
        g = torch.zeros_like(self.w)
        for L, lv in enumerate(leaves):
            o = self.off[L]
            for name, shp in self.spec.layer_segments(L):
                k = int(np.prod(shp))
                if lv[name].grad is not None:
                    g[o:o + k] = lv[name].grad.reshape(-1)
                o += k
        del leaves, base
        self.t += 1
        self.m.lerp_(g, 1 - self.b1)
        self.v.mul_(self.b2).addcmul_(g, g, value=1 - self.b2)
        bc1 = 1 - self.b1 ** self.t
        bc2 = 1 - self.b2 ** self.t
        denom = (self.v.sqrt() / math.sqrt(bc2)).add_(self.eps)
        self.w.addcdiv_(self.m, denom, value=-self.lr / bc1)
        return total / n
