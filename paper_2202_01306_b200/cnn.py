"""Deep-CNN layer chains (BASELINE config c5: VGG-416 / ResNet-1026-style
layer packs) as the runtime lays them out, and the ProfileSet generated from
their real tensor shapes.

A chain layer is one of (``include/harmony_b200.h`` hm_cnn_layer):

* ``conv``: 3x3 convolution (stride 1, zero padding 1) + bias + ReLU;
* ``down``: the same, then a 2x2 average pool (stage transition);
* ``res``:  basic residual block ``relu(x + conv2(relu(conv1(x))))``;
* ``head``: global average pool + fully connected classifier + cross-entropy;
* ``res2``: the second half of a residual block at convolution granularity,
  ``relu(conv(x) + skip)``, where skip is the output of an earlier layer.

With whole-block ``res`` layers the chain is linear: pack boundaries carry one
tensor each and the schedule needs no relays (``core.py:181-265``). With
``res2`` layers (``cnn_chain(kind="fine")``, one chain node per convolution,
as the paper decomposes ResNet-1026) the skip edge can cross pack boundaries.
``CNNSpec.chain()`` serializes the layer DAG with the reference's relays
(``serialize_graph``). The runtime keeps skip tensors and their gradients in
device-resident relay stores; they are SHARED_MEMORY hand-offs, so the ledger
bills no bytes for them.

Deviations from torchvision VGG / ResNet, kept in the CPU oracle too:

* no BatchNorm, because per-microbatch statistics would make the loss depend on
  the microbatch size u, which Harmony's equivalence to single-device
  training (``PAPER.md:521-523``) forbids;
* residual branches are initialised small (SkipInit-style) so the chain stays
  trainable at depth;
* 2x2 average pooling instead of stride-2 convolutions;
* images enter zero-padded to 64 channels, because the implicit-GEMM
  convolution gathers 64-channel slices.

Byte model (what the swap engine moves):

* W(L) = 4 B x params(L);
* dW(L) = W(L);
* K(L) = 8 B x params(L);
* x(L, u) = u * h * w * cin * 2, the NHWC bf16 activation entering layer L;
* y(L, u) = x(L + 1, u).

The head's y is defined as its own x; it is only billed for Harmony-PP seams,
which the CNN runtime keeps on one GPU.
"""

from __future__ import annotations

from dataclasses import dataclass

from .profiler import AffineModel, ProfileSet

CONV, DOWN, RES, HEAD, RES2 = 0, 1, 2, 3, 4
_TYPES = {"conv": CONV, "down": DOWN, "res": RES, "head": HEAD, "res2": RES2}


def _pad64(v: int) -> int:
    return -(-v // 64) * 64


@dataclass(frozen=True)
class CNNSpec:
    """layers: ((type, cin, cout, h, w), ...) with (h, w, cin) the layer input."""
    layers: tuple[tuple[int, int, int, int, int], ...]
    classes: int
    name: str = "cnn"
    skips: tuple[int, ...] = ()  # per layer: source layer of a res2's skip input, -1 otherwise

    def __post_init__(self) -> None:
        R = len(self.layers)
        if not self.skips:
            object.__setattr__(self, "skips", (-1,) * R)
        if len(self.skips) != R:
            raise ValueError("one skip entry per layer")
        for L, src in enumerate(self.skips):
            t, cin, cout, h, w = self.layers[L]
            if (t == RES2) != (src >= 0):
                raise ValueError(f"layer {L}: exactly the res2 layers have a skip source")
            if t == RES2:
                if not 0 <= src < L - 1 or cin != cout:
                    raise ValueError(f"layer {L}: res2 needs an earlier skip source and equal widths")
                st, _, scout, sh, sw = self.layers[src]
                oh, ow = (sh // 2, sw // 2) if st == DOWN else (sh, sw)
                if (scout, oh, ow) != (cout, h, w):
                    raise ValueError(f"layer {L}: skip source {src} has a different shape")
        if R < 1 or self.layers[-1][0] != HEAD or any(t == HEAD for t, *_ in self.layers[:-1]):
            raise ValueError("a CNN chain ends with exactly one head layer")
        for L, (t, cin, cout, h, w) in enumerate(self.layers):
            if cin % 64 or (t != HEAD and cout % 64):
                raise ValueError(f"layer {L}: channels must be multiples of 64")
            if t == RES and cin != cout:
                raise ValueError(f"layer {L}: residual blocks keep the width")
            if L + 1 < R:
                nt, ncin, _, nh, nw = self.layers[L + 1]
                oh, ow = (h // 2, w // 2) if t == DOWN else (h, w)
                if (ncin, nh, nw) != (cout, oh, ow):
                    raise ValueError(f"layer {L}: output shape does not feed layer {L + 1}")

    @property
    def n_layer(self) -> int:
        return len(self.layers)

    @property
    def classes_padded(self) -> int:
        return _pad64(self.classes)

    @property
    def image(self) -> tuple[int, int, int]:
        _, cin, _, h, w = self.layers[0]
        return h, w, cin

    # -- parameters --------------------------------------------------------
    def layer_segments(self, L: int) -> list[tuple[str, tuple[int, ...]]]:
        """Ordered (name, shape) of layer L's parameters in the W arena (weights
        [cout, 3, 3, cin], the layout the implicit-GEMM convolution reads)."""
        t, cin, cout, _, _ = self.layers[L]
        if t == HEAD:
            return [("w1", (self.classes_padded, cin)), ("b1", (self.classes_padded,))]
        seg = [("w1", (cout, 3, 3, cin)), ("b1", (cout,))]
        if t == RES:  # (res2 is one convolution: w1, b1)
            seg += [("w2", (cout, 3, 3, cout)), ("b2", (cout,))]
        return seg

    def layer_params(self, L: int) -> int:
        n = 0
        for _, shp in self.layer_segments(L):
            k = 1
            for s in shp:
                k *= s
            n += k
        return n

    def total_params(self) -> int:
        return sum(self.layer_params(L) for L in range(self.n_layer))

    # -- bytes / FLOPs -----------------------------------------------------
    def x_bytes(self, L: int) -> int:
        """Per-sample bytes of the bf16 NHWC tensor entering layer L."""
        if L >= self.n_layer:
            return self.x_bytes(self.n_layer - 1)
        _, cin, _, h, w = self.layers[L]
        return h * w * cin * 2

    def layer_fwd_flops(self, L: int, u: int) -> int:
        t, cin, cout, h, w = self.layers[L]
        if t == HEAD:
            return 2 * u * cin * self.classes
        f = 2 * u * h * w * 9 * cin * cout
        return 2 * f if t == RES else f  # res2: one convolution

    def act_bytes_per_sample(self, L: int) -> int:
        t, cin, cout, h, w = self.layers[L]
        if t == HEAD:
            return 2 * cin + 2 * self.classes_padded
        y = h * w * cout * 2
        return {CONV: y, DOWN: y + y // 4, RES: 2 * y, RES2: y}[t] + h * w * cin * 2

    def chain(self):
        """The planner's LayerChain: the layer DAG (skip edges included)
        serialized with the reference's relay annotations (``core.py:181-265``)."""
        from .core import LayerChain, LayerNode, serialize_graph
        if all(s < 0 for s in self.skips):
            return LayerChain.linear(self.n_layer)
        nodes = [LayerNode(L, predecessors=tuple(p for p in ((L - 1,) if L else ()) + ((self.skips[L],)
                                                                                        if self.skips[L] >= 0 else ())))
                 for L in range(self.n_layer)]
        return serialize_graph(nodes)


def cnn_chain(name: str, image: int, widths: list[int], blocks: list[int], classes: int, kind: str = "res",
              stem_downs: int = 0) -> CNNSpec:
    """Stem conv (+ ``stem_downs`` down layers of the first width), then per
    stage ``blocks[s]`` res blocks (kind "res") or conv layers (kind "vgg") of
    width ``widths[s]``, a ``down`` layer between stages, and the head."""
    layers, skips = [], []
    h = image
    cin = 64  # the image, zero-padded to 64 channels
    layers.append((CONV, cin, widths[0], h, h))
    skips.append(-1)
    cin = widths[0]
    for _ in range(stem_downs):
        layers.append((DOWN, cin, widths[0], h, h))
        skips.append(-1)
        h //= 2
    for s, (wd, nb) in enumerate(zip(widths, blocks)):
        for _ in range(nb):
            if kind == "fine":  # one chain node per convolution; the skip spans the pair
                if cin != wd:
                    raise ValueError("fine residual stages keep the width (use a down layer between stages)")
                src = len(layers) - 1
                layers.append((CONV, cin, wd, h, h))
                layers.append((RES2, wd, wd, h, h))
                skips += [-1, src]
            else:
                layers.append((RES if kind == "res" else CONV, cin, wd, h, h))
                skips.append(-1)
            cin = wd
        if s + 1 < len(widths):
            layers.append((DOWN, cin, widths[s + 1], h, h))
            skips.append(-1)
            cin = widths[s + 1]
            h //= 2
    layers.append((HEAD, cin, 0, h, h))
    skips.append(-1)
    return CNNSpec(tuple(layers), classes, name, tuple(skips))


CNN_PRESETS = {
    # small chains for parity tests (16x16 images, 10 classes)
    "resnet-tiny": cnn_chain("resnet-tiny", 16, [64, 128], [2, 2], 10, "res"),
    "vgg-tiny": cnn_chain("vgg-tiny", 16, [64, 128], [2, 2], 10, "vgg"),
    # convolution-granularity residual chain: skip edges cross pack boundaries (relays)
    "resnet-fine-tiny": cnn_chain("resnet-fine-tiny", 16, [64, 128], [2, 2], 10, "fine"),
    # BASELINE config c5 shapes at 224^2 / 1000 classes (stem, two stem downs to
    # 56^2, stages at 56/28/14/7): ResNet-1026 = 1 + 2 + 2 x 510 + 3 = 1026
    # convolutions + classifier; VGG-416 = 1 + 2 + 410 + 3 = 416 convolutions
    # (four stages: a fifth would pool the 7^2 maps)
    "resnet-1026": cnn_chain("resnet-1026", 224, [64, 128, 256, 512], [128, 128, 128, 126], 1000, "res", 2),
    "vgg-416": cnn_chain("vgg-416", 224, [64, 128, 256, 512], [103, 103, 103, 101], 1000, "vgg", 2),
    # one-GPU bench workload: ResNet-style, 56x56, 128 blocks
    "resnet-bench": cnn_chain("resnet-bench", 56, [128, 256], [64, 62], 1000, "res"),
}


def cnn_profiles(spec: CNNSpec, u_max: int = 64, tflops: float = 1.0e15, hbm_gbs: float = 6.5e12,
                 measured: dict | None = None) -> ProfileSet:
    """ProfileSet from the real shapes (bytes exact, times FLOP-derived or
    fitted), same construction as ``model.gpt_profiles``."""
    R = spec.n_layer
    tm, mm, xm, ym, w, dw, k = {}, {}, {}, {}, {}, {}, {}
    for L in range(R):
        p = spec.layer_params(L)
        w[L], dw[L], k[L] = 4 * p, 4 * p, 8 * p
        xm[L] = AffineModel(float(spec.x_bytes(L)), 0.0)
        ym[L] = AffineModel(float(spec.x_bytes(L + 1)), 0.0)
        f1 = spec.layer_fwd_flops(L, 1) / tflops * 1e9
        if measured and (L, "F") in measured:
            tm[(L, "F")] = AffineModel(*measured[(L, "F")])
            tm[(L, "B")] = AffineModel(*measured[(L, "B")])
        else:
            tm[(L, "F")] = AffineModel(f1, 0.0)
            tm[(L, "B")] = AffineModel(2 * f1, 0.0)
        tm[(L, "U")] = AffineModel(0.0, 28 * p / hbm_gbs * 1e9)
        act = float(spec.act_bytes_per_sample(L))
        mm[(L, "F")] = AffineModel(act, float(w[L] * 3 // 2))
        mm[(L, "B")] = AffineModel(act, float(w[L] * 3 // 2 + dw[L]))
        mm[(L, "U")] = AffineModel(0.0, float(w[L] + dw[L] + k[L]))
    return ProfileSet(R, tm, mm, xm, ym, w, dw, k, u_max_f=u_max, u_max_b=u_max)


def synthetic_images(spec: CNNSpec, samples: int, seed: int = 1234):
    """Synthetic minibatch: images N(0, 1) with 3 real channels, zero-padded to
    64 (NHWC bf16, returned as a torch tensor), labels uniform in [0, classes)
    from torch.Generator().manual_seed(seed)."""
    import torch
    g = torch.Generator().manual_seed(seed)
    h, w, c = spec.image
    img = torch.zeros(samples, h, w, c, dtype=torch.float32)
    img[..., :3] = torch.randn(samples, h, w, 3, generator=g)
    labels = torch.randint(0, spec.classes, (samples,), generator=g, dtype=torch.int32)
    return img.to(torch.bfloat16).contiguous(), labels.contiguous()
