"""GPT / BERT-style layer chain as the runtime lays it out, and the
ProfileSet generated from its real tensor shapes.

Layer L of the chain is one transformer block; the token + position
embedding is fused into layer 0 and the final LayerNorm + LM head +
cross-entropy into layer R-1.  Embedding and head are
untied because the per-layer W model cannot express tying
(`profiler.py:163-167`).

Byte model (every number the swap engine moves; fp32 master state):
* W(L)  = 4 B x params(L)           -- master weights, swapped per task
* dW(L) = W(L)                      -- GPU-resident grad buffer, never swapped
* K(L)  = 8 B x params(L)           -- Adam (m, v) interleaved per parameter
* x(L, u) = u*s*d*4 for L >= 1      -- fp32 residual stream entering block L
* x(0, u) = u*s*4                   -- int32 token ids entering the embedding
* y(L, u) = u*s*d*4                 -- fp32 residual stream leaving block L
The LM head's vocabulary is padded to a multiple of 128 so every row stride
is 16-byte aligned for TMA; the padding is part of W(R-1).
"""

from __future__ import annotations

from dataclasses import dataclass

from .core import MachineModel
from .profiler import AffineModel, ProfileSet


def pad_vocab(v: int, multiple: int = 128) -> int:
    return -(-v // multiple) * multiple


@dataclass(frozen=True)
class GPTSpec:
    n_layer: int
    d_model: int
    n_head: int
    seq_len: int
    vocab: int
    causal: bool = True
    name: str = "gpt"

    def __post_init__(self) -> None:
        if self.d_model % self.n_head:
            raise ValueError("d_model must be divisible by n_head")
        if self.head_dim not in (64, 128):
            raise ValueError("head_dim must be 64 or 128 (attention kernel tiles)")
        if self.d_model % 64:
            raise ValueError("d_model must be a multiple of 64")
        if self.seq_len % 64:
            raise ValueError("seq_len must be a multiple of 64")

    @property
    def head_dim(self) -> int:
        return self.d_model // self.n_head

    @property
    def vocab_padded(self) -> int:
        return pad_vocab(self.vocab)

    # -- parameters --------------------------------------------------------
    def block_params(self) -> int:
        d = self.d_model
        return 12 * d * d + 13 * d

    def embed_params(self) -> int:
        return (self.vocab_padded + self.seq_len) * self.d_model

    def head_params(self) -> int:
        return 2 * self.d_model + self.vocab_padded * self.d_model

    def layer_params(self, L: int) -> int:
        p = self.block_params()
        if L == 0:
            p += self.embed_params()
        if L == self.n_layer - 1:
            p += self.head_params()
        return p

    def total_params(self) -> int:
        return sum(self.layer_params(L) for L in range(self.n_layer))

    def layer_segments(self, L: int) -> list[tuple[str, int]]:
        """Ordered (name, numel) of layer L's parameters in the W arena."""
        d, v, s = self.d_model, self.vocab_padded, self.seq_len
        # parameters read in fp32 (LayerNorm, biases, embedding tables) first,
        # then the GEMM weights: the fp32 prefix is what a forward task needs
        # beyond the bf16 high halves in the bf16 swap-payload mode
        seg = [("ln1_g", d), ("ln1_b", d), ("b_qkv", 3 * d), ("b_proj", d), ("ln2_g", d), ("ln2_b", d),
               ("b_fc1", 4 * d), ("b_fc2", d)]
        if L == self.n_layer - 1:
            seg += [("lnf_g", d), ("lnf_b", d)]
        if L == 0:
            seg += [("wte", v * d), ("wpe", s * d)]
        seg += [("w_qkv", 3 * d * d), ("w_proj", d * d), ("w_fc1", 4 * d * d), ("w_fc2", 4 * d * d)]
        if L == self.n_layer - 1:
            seg += [("w_head", v * d)]
        return seg

    def f32_prefix(self, L: int) -> int:
        """Leading parameters of layer L that kernels read in fp32."""
        n = 0
        for name, k in self.layer_segments(L):
            if name.startswith("w_"):
                break
            n += k
        return n

    # -- FLOPs (BASELINE.md "Algorithmic FLOPs") ----------------------------
    def layer_fwd_flops(self, L: int, u: int) -> int:
        s, d = self.seq_len, self.d_model
        f = u * s * (24 * d * d + 4 * s * d)
        if L == self.n_layer - 1:
            f += 2 * u * s * d * self.vocab
        return f

    # -- activations kept per sample for backward (bytes) -------------------
    def act_bytes_per_sample(self, L: int) -> int:
        s, d, h = self.seq_len, self.d_model, self.n_head
        per_tok = (4 * d        # x fp32 (block input)
                   + 2 * d      # ln1 out bf16
                   + 8          # mean/rstd
                   + 2 * 3 * d  # qkv bf16
                   + 2 * d      # attention out bf16
                   + 4 * h      # lse fp32
                   + 4 * d      # h1 fp32
                   + 2 * d + 8  # ln2 out + stats
                   + 2 * 4 * d  # fc1 pre-activation bf16
                   + 2 * 4 * d)  # gelu out bf16
        b = s * per_tok
        if L == self.n_layer - 1:
            b += s * (4 * d + 2 * d + 8 + 2 * self.vocab_padded)  # block out, lnf out, stats, dlogits
        return b


GPT_PRESETS = {
    # c1: tiny GPT-2: 4 layers, d=256, 4 heads, seq 128, V=1024
    "tiny": GPTSpec(4, 256, 4, 128, 1024, True, "tiny-gpt2"),
    # c2: BERT-Large shapes (full attention)
    "bert-large": GPTSpec(24, 1024, 16, 512, 30522, False, "bert-large"),
    # c3: GPT-2 XL 1.5B
    "gpt2-xl": GPTSpec(48, 1600, 25, 1024, 50257, True, "gpt2-xl"),
    # c4: GPT-style 40B
    "gpt-40b": GPTSpec(48, 8192, 64, 1024, 50257, True, "gpt-40b"),
    # c4's layer shape at the largest depth one box's host RAM (197 GiB) can pin:
    # 15.3 B params, W + Adam state = 184 GB > 180 GB HBM (W + dW + K = 245 GB)
    "gpt-15b": GPTSpec(18, 8192, 64, 1024, 50257, True, "gpt-15b"),
}


def gpt_profiles(spec: GPTSpec, u_max: int = 64, tflops: float = 1.0e15,
                 hbm_gbs: float = 6.5e12, measured: dict | None = None) -> ProfileSet:
    """ProfileSet from real shapes.  Times are FLOP / ``tflops`` (F), 2x (B)
    and the Adam stream time 28 B/param / ``hbm_gbs`` (U) unless ``measured``
    supplies fitted (slope, intercept) per (layer, pass)."""
    R = spec.n_layer
    tm, mm, xm, ym, w, dw, k = {}, {}, {}, {}, {}, {}, {}
    sd4 = spec.seq_len * spec.d_model * 4
    for L in range(R):
        p = spec.layer_params(L)
        w[L] = 4 * p
        dw[L] = 4 * p
        k[L] = 8 * p
        xm[L] = AffineModel(float(spec.seq_len * 4 if L == 0 else sd4), 0.0)
        ym[L] = AffineModel(float(sd4), 0.0)
        f1 = spec.layer_fwd_flops(L, 1) / tflops * 1e9
        if measured and (L, "F") in measured:
            tm[(L, "F")] = AffineModel(*measured[(L, "F")])
            tm[(L, "B")] = AffineModel(*measured[(L, "B")])
        else:
            tm[(L, "F")] = AffineModel(f1, 0.0)
            tm[(L, "B")] = AffineModel(2 * f1, 0.0)
        tm[(L, "U")] = AffineModel(0.0, 28 * p / hbm_gbs * 1e9)
        act = float(spec.act_bytes_per_sample(L))
        mm[(L, "F")] = AffineModel(act, float(w[L] * 3 // 2))  # fp32 W + bf16 shadow
        mm[(L, "B")] = AffineModel(act, float(w[L] * 3 // 2 + dw[L]))
        mm[(L, "U")] = AffineModel(0.0, float(w[L] + dw[L] + k[L]))
    return ProfileSet(R, tm, mm, xm, ym, w, dw, k, u_max_f=u_max, u_max_b=u_max)


def gpt_machine(gpu_count: int = 1, alpha_bytes: int = 160 << 30,
                pcie_gbs: float = 55e9, nvlink_gbs: float = 770e9, root_gbs: float = 0.0) -> MachineModel:
    """B200 server model: measured PCIe Gen5 x16 per direction, one NVSwitch
    group, NVLink peer bandwidth."""
    return MachineModel(gpu_count=gpu_count, gpu_mem_capacity=int(alpha_bytes),
                        pcie_bandwidth=int(pcie_gbs), root_link_bandwidth=int(root_gbs),
                        p2p_bandwidth=int(nvlink_gbs))


def synthetic_batch(spec: GPTSpec, samples: int, seed: int = 1234):
    """Synthetic minibatch: tokens i.i.d. uniform in [0, V)
    from torch.Generator().manual_seed(seed); labels = tokens shifted by one."""
    import numpy as np
    import torch
    g = torch.Generator().manual_seed(seed)
    seq = torch.randint(0, spec.vocab, (samples, spec.seq_len + 1), generator=g, dtype=torch.int64)
    return (np.ascontiguousarray(seq[:, :-1].numpy().astype(np.int32)),
            np.ascontiguousarray(seq[:, 1:].numpy().astype(np.int32)))


# -- bf16 swap payloads: exact split of fp32 weights ------------
def split_planes(w):
    """fp32 -> (hi, lo) uint16 planes: hi = bf16 nearest with ties toward zero
    ((bits + 0x7FFF) >> 16, the GEMM operand), lo = the low 16 bits."""
    import numpy as np
    u = np.ascontiguousarray(w, dtype=np.float32).view(np.uint32).reshape(-1)
    hi = np.empty(u.size, np.uint16)
    lo = np.empty(u.size, np.uint16)
    step = 1 << 24  # bounded temporaries (a 15 B-parameter arena leaves little host RAM)
    for i in range(0, u.size, step):
        c = u[i:i + step]
        # uint32 wrap-around only for NaN bit patterns >= 0xFFFF8001
        hi[i:i + step] = (c + np.uint32(0x7FFF)) >> np.uint32(16)
        lo[i:i + step] = c & np.uint32(0xFFFF)
    return hi, lo


def join_planes(hi, lo):
    """Inverse of split_planes, bit-exact: bits = (hi << 16) + d with d = lo for
    lo <= 0x8000, else lo - 0x10000."""
    import numpy as np
    out = np.empty(hi.size, np.uint32)
    step = 1 << 24
    for i in range(0, hi.size, step):
        h = hi[i:i + step].astype(np.uint32)
        l_ = lo[i:i + step].astype(np.uint32)
        # (h << 16) + d, d = lo or lo - 0x10000: modulo 2^32 the same as subtracting 0x10000 from h << 16
        out[i:i + step] = (h << np.uint32(16)) + l_ - np.where(l_ > 0x8000, np.uint32(0x10000), np.uint32(0))
    return out.view(np.float32)
