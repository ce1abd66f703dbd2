"""``execute``: run a task graph on the GPU through the native runtime.

Drop-in sibling of :func:`paper_2202_01306_b200.simulator.simulate`
(`pkg/src/wrapsched/simulator.py:378-434` is the reference's estimate of the
same iteration).  The returned ``SimReport`` is built from CUDA events of the
executed iteration; its ledger rows, byte volumes and per-GPU volumes equal
``simulate``'s because the runtime executes the same native plan.

One ``HarmonyRuntime`` per process and GPU.  Model state lives in the
runtime's pinned host arenas (W fp32, K = Adam (m, v) interleaved): the GPU
only ever holds the packs the schedule swaps in.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as NL
from .core import MachineModel, gpu_shares
from .errors import ValidationError
from .lowering import NativePlan
from .cnn import CNNSpec
from .model import GPTSpec, join_planes, split_planes
from .profiler import ProfileSet
from .simulator import SimReport, report_from_items
from .taskgraph import TaskGraph


class HarmonyRuntime:
    """Native runtime for one GPU: arenas, streams, kernels, plan executor."""

    def __init__(self, spec: GPTSpec | CNNSpec, *, alpha_bytes: int, device: int = 0, lr: float = 1e-4,
                 betas: tuple[float, float] = (0.9, 0.999), eps: float = 1e-8, w_payload: str = "fp32",
                 math: str = "bf16", dp_update: str = "replicated") -> None:
        """``w_payload``: "fp32" swaps fp32 W exactly as the reference's ledger
        bills it; "bf16" is the SURVEY 8f4b fast mode (transformer family): the
        host W arena holds each layer as [bf16 hi plane | 16-bit lo plane], an
        exact split of the fp32 value, and forward tasks move only the hi plane
        plus the lo plane of the fp32-read prefix (LayerNorm, biases,
        embeddings).  Losses and weights are bit-identical to "fp32"; the
        forward W rows of the ledger differ (flagged: not the reference's).

        ``math``: "bf16" = bf16 tensor-core operands with fp32 accumulation
        (the throughput mode); "fp32" = the parity mode (transformer family):
        fp32 activations, GEMMs as three-plane bf16 split products on the same
        tcgen05 kernel, fp32 attention (DESIGN.md section 6 states both
        modes' tolerances).  The swap plan and ledger are the same.

        ``dp_update`` (Harmony-DP only): "replicated" is the reference -- every
        rank keeps its own host replica of W and K and updates every pack;
        "sharded" is the SURVEY 8f row-4 fast mode -- one host arena shared by
        all ranks (``share_arenas``), gradients reduce-scattered, rank g
        updates, swaps in and swaps out only shard g of each pack's K and W
        (hm_machine.dp_sharded_update states the split).  Per GPU that moves
        2|W| + 5|W|/N instead of 7|W| (Adam fp32) and holds one host copy
        instead of N; the U rows of the ledger differ from the reference at
        N > 1 (flagged; ``simulate(..., dp_update="sharded")`` prices it)."""
        if dp_update not in ("replicated", "sharded"):
            raise ValidationError("dp_update must be 'replicated' or 'sharded'")
        if dp_update == "sharded" and w_payload != "fp32":
            raise ValidationError("the sharded update and bf16 W payloads are exclusive")
        self.dp_update = dp_update
        if w_payload not in ("fp32", "bf16"):
            raise ValidationError("w_payload must be 'fp32' or 'bf16'")
        if math not in ("bf16", "fp32"):
            raise ValidationError("math must be 'bf16' or 'fp32'")
        if math == "fp32" and (isinstance(spec, CNNSpec) or w_payload == "bf16"):
            raise ValidationError("math='fp32' is implemented for the transformer family with fp32 W payloads")
        self.spec = spec
        self.w_payload = w_payload
        self.math = math
        self.hparams = (float(lr), float(betas[0]), float(betas[1]), float(eps))
        self.lib = NL.lib()
        self.is_cnn = isinstance(spec, CNNSpec)
        st = C.c_int32(0)
        if self.is_cnn:
            arr = (NL.hm_cnn_layer * spec.n_layer)(*[NL.hm_cnn_layer(*lay, sk)
                                                      for lay, sk in zip(spec.layers, spec.skips)])
            m = NL.hm_cnn_model(spec.n_layer, arr, spec.classes, spec.classes_padded, lr, betas[0], betas[1], eps)
            self._model = (m, arr)
            h = self.lib.hm_runtime_create_cnn(device, C.byref(m), int(alpha_bytes), C.byref(st))
        else:
            m = NL.hm_model(spec.n_layer, spec.d_model, spec.n_head, spec.seq_len, spec.vocab,
                            spec.vocab_padded, 1 if spec.causal else 0, 1 if math == "fp32" else 0,
                            lr, betas[0], betas[1], eps)
            self._model = m
            h = self.lib.hm_runtime_create(device, C.byref(m), int(alpha_bytes), C.byref(st))
        if not h:
            NL.check(st.value or -4)
        self.handle = h
        self.alpha_bytes = int(alpha_bytes)
        offs = (C.c_int64 * (spec.n_layer + 1))()
        NL.check(self.lib.hm_runtime_layer_offsets(h, offs, spec.n_layer + 1))
        self.w_off = np.array(offs[:], dtype=np.int64)
        for L in range(spec.n_layer):
            if self.w_off[L + 1] - self.w_off[L] != spec.layer_params(L):
                raise ValidationError(f"native layout of layer {L} disagrees with GPTSpec")
        if w_payload == "bf16":
            if self.is_cnn:
                raise ValidationError("bf16 W payloads are implemented for the transformer family")
            NL.check(self.lib.hm_runtime_set_w_payload(h, 1))
        self._w_arena = self._arena(0, np.float32)
        self.k = self._arena(1, np.float32)
        self.plan: NativePlan | None = None
        self.graph: TaskGraph | None = None
        self.rank = 0
        self.samples = 0
        self.device = device
        self._checked: tuple | None = None  # (ptr, version) of the last range-checked CUDA inputs

    def _arena(self, kind: int, dtype) -> np.ndarray:
        nbytes = C.c_int64(0)
        ptr = self.lib.hm_runtime_arena(self.handle, kind, C.byref(nbytes))
        n = nbytes.value // np.dtype(dtype).itemsize
        return np.ctypeslib.as_array(C.cast(ptr, C.POINTER(C.c_float)), shape=(n,))

    # -- state ----------------------------------------------------------------
    @property
    def w(self) -> np.ndarray:
        """Master weights, canonical fp32 layout: the W arena itself (fp32
        payload) or a decoded copy of its planes (bf16 payload)."""
        return self._w_arena if self.w_payload == "fp32" else self.weights()

    def weights(self) -> np.ndarray:
        """Copy of the master weights in the canonical fp32 layout."""
        if self.w_payload == "fp32":
            return self._w_arena.copy()
        a16 = self._w_arena.view(np.uint16)
        out = np.empty(self._w_arena.size, dtype=np.float32)
        for L in range(self.spec.n_layer):
            o, n = int(self.w_off[L]), int(self.w_off[L + 1] - self.w_off[L])
            out[o:o + n] = join_planes(a16[2 * o:2 * o + n], a16[2 * o + n:2 * o + 2 * n])
        return out

    def set_weights(self, flat: np.ndarray) -> None:
        """Write canonical fp32 master weights into the W arena (bf16 payload:
        as per-layer [hi | lo] planes, hi = nearest bf16 with ties toward zero,
        lo = the low 16 bits; the split is exact)."""
        flat = np.ascontiguousarray(flat, dtype=np.float32)
        if flat.size != self._w_arena.size:
            raise ValidationError("weights size disagrees with the model")
        if self.w_payload == "fp32":
            self._w_arena[:] = flat
            return
        for L in range(self.spec.n_layer):
            self._set_layer(L, flat[int(self.w_off[L]):int(self.w_off[L + 1])])

    def w_fwd_bytes(self) -> list[int] | None:
        """Per-layer W bytes a forward task moves (bf16 payload), else None."""
        if self.w_payload == "fp32":
            return None
        return [2 * self.spec.layer_params(L) + 2 * self.spec.f32_prefix(L) for L in range(self.spec.n_layer)]

    def _segment_views(self, L: int, buf: np.ndarray) -> dict[str, np.ndarray]:
        """Views of layer L's segments in a layer-sized canonical buffer."""
        out, o = {}, 0
        for name, shp in self.spec.layer_segments(L):
            n = int(np.prod(shp)) if isinstance(shp, tuple) else int(shp)
            out[name] = buf[o:o + n].reshape(shp) if isinstance(shp, tuple) else buf[o:o + n]
            o += n
        return out

    def _set_layer(self, L: int, buf: np.ndarray) -> None:
        o, n = int(self.w_off[L]), int(self.w_off[L + 1] - self.w_off[L])
        a16 = self._w_arena.view(np.uint16)
        a16[2 * o:2 * o + n], a16[2 * o + n:2 * o + 2 * n] = split_planes(buf)

    def layer_params(self, L: int, base: np.ndarray | None = None) -> dict[str, np.ndarray]:
        """Views of layer L's master weights, by segment name (CNN segments
        come shaped: weights [cout, 3, 3, cin]), in ``base`` (a canonical
        flat array) or the W arena itself (fp32 payload only)."""
        if base is None:
            if self.w_payload != "fp32":
                raise ValidationError("bf16 W payload: read weights() / write set_weights()")
            base = self._w_arena
        out, o = {}, int(self.w_off[L])
        for name, shp in self.spec.layer_segments(L):
            n = int(np.prod(shp)) if isinstance(shp, tuple) else int(shp)
            out[name] = base[o:o + n].reshape(shp) if isinstance(shp, tuple) else base[o:o + n]
            o += n
        return out

    def _init_cnn(self, seed: int) -> None:
        """He-normal convolutions (fan-in 9 x the real input channels), the
        second convolution of a residual block scaled by 0.1 (SkipInit-style:
        no BatchNorm), classifier N(0, 0.01) with zero padding rows, zero
        biases; Adam state zero."""
        import torch
        from .cnn import HEAD, RES
        gen = torch.Generator().manual_seed(seed)
        for L, (t, cin, cout, _, _) in enumerate(self.spec.layers):
            p = self.layer_params(L)
            for name, view in p.items():
                if name.startswith("b"):
                    view[...] = 0.0
                    continue
                shape = tuple(view.shape)
                if t == HEAD:
                    v = torch.empty(shape).normal_(0.0, 0.01, generator=gen)
                    v[self.spec.classes:] = 0.0
                else:
                    fan_in = 9 * (3 if L == 0 else shape[-1])
                    v = torch.empty(shape).normal_(0.0, (2.0 / fan_in) ** 0.5, generator=gen)
                    if L == 0:
                        v[..., 3:] = 0.0  # padded image channels
                    if t == RES and name == "w2":
                        v *= 0.1
                view[...] = v.numpy()
        self.k[:] = 0.0

    def init_weights(self, seed: int = 0, device: str | None = None) -> None:
        """N(0, 0.02) matrices/embeddings, LayerNorm gamma=1 / beta=0, zero
        biases, zero padded vocabulary rows; Adam state zero.
        ``device="cuda"`` draws the normals on the GPU and copies them into the
        pinned arena (seconds instead of minutes for a 15 B-parameter model;
        a different random stream than the CPU generator)."""
        import torch
        if self.is_cnn:
            return self._init_cnn(seed)
        V, d = self.spec.vocab, self.spec.d_model
        gen = torch.Generator(device=device).manual_seed(seed) if device is not None else \
            torch.Generator().manual_seed(seed)
        for L in range(self.spec.n_layer):
            # one layer at a time: the W arena itself (fp32 payload) or a layer-sized
            # canonical buffer split into the arena's planes (bf16 payload)
            o, n = int(self.w_off[L]), int(self.w_off[L + 1] - self.w_off[L])
            buf = self._w_arena[o:o + n] if self.w_payload == "fp32" else np.empty(n, np.float32)
            for name, view in self._segment_views(L, buf).items():
                if name.endswith("_g"):
                    view[:] = 1.0
                elif name.startswith("b_") or name.endswith("_b"):
                    view[:] = 0.0
                elif device is not None:
                    t = torch.empty(view.size, dtype=torch.float32, device=device).normal_(0.0, 0.02, generator=gen)
                    if name in ("wte", "w_head"):
                        t.view(-1, d)[V:] = 0.0
                    torch.from_numpy(view).copy_(t)
                    del t
                else:
                    t = torch.empty(view.size, dtype=torch.float32).normal_(0.0, 0.02, generator=gen)
                    view[:] = t.numpy()
                    if name in ("wte", "w_head"):
                        view.reshape(-1, d)[V:] = 0.0
            if self.w_payload != "fp32":
                self._set_layer(L, buf)
        if device is None:
            self.k[:] = 0.0  # (hm_runtime_create zeroes K; kept for re-initialisation)

    # -- checkpoint / resume (the host arenas are the model state) ------
    def _fingerprint(self) -> np.ndarray:
        """Model identity stored with a checkpoint: the family's shape fields
        (CNN: every layer's (type, cin, cout, h, w, skip) and the classes)."""
        sp = self.spec
        if self.is_cnn:
            rows = [list(lay) + [sk] for lay, sk in zip(sp.layers, sp.skips)]
            return np.array([1, sp.n_layer, sp.classes] + [v for r in rows for v in r], dtype=np.int64)
        return np.array([0, sp.n_layer, sp.d_model, sp.n_head, sp.seq_len, sp.vocab, int(sp.causal)],
                        dtype=np.int64)

    def save_checkpoint(self, path: str) -> None:
        """W and K arenas + optimizer step and hyperparameters, as one .npz (no
        device state: the GPU only holds transient packs between iterations).
        W is stored in the canonical fp32 layout whatever the payload mode."""
        np.savez(path, w=self.weights(), k=self.k, step=np.int64(self.lib.hm_runtime_get_step(self.handle)),
                 spec=self._fingerprint(), hparams=np.array(self.hparams, dtype=np.float64))
        return None

    def load_checkpoint(self, path: str) -> None:
        z = np.load(path)
        if not np.array_equal(z["spec"], self._fingerprint()) or z["w"].shape != (int(self.w_off[-1]),):
            raise ValidationError("checkpoint was written for a different model")
        if "hparams" in z and not np.array_equal(z["hparams"], np.array(self.hparams, dtype=np.float64)):
            raise ValidationError(f"checkpoint optimizer hyperparameters {tuple(z['hparams'])} differ from this "
                                  f"runtime's {self.hparams} (resume would not be exact)")
        self.set_weights(z["w"])
        self.k[:] = z["k"]
        NL.check(self.lib.hm_runtime_set_step(self.handle, int(z["step"])))

    # -- Harmony-PP across processes ----------------------------------------------
    @staticmethod
    def stash_bytes_for(graph: TaskGraph, profiles: ProfileSet) -> int:
        """Host stash arena size the native layout needs (one region per
        backward-pack head, D samples, 4 KiB aligned)."""
        heads = sorted({L for t in graph.tasks for k, e in t.outputs.items() if k.value == "sX" for L in e})
        return sum(-(-profiles.x_bytes(L, graph.minibatch) // 4096) * 4096 for L in heads)

    def share_arenas(self, name: str, create: bool, stash_bytes: int) -> None:
        """Move W / K / stash into one shared-memory segment (every PP rank
        maps the same pinned host state).  Rank 0 creates, the others attach."""
        NL.check(self.lib.hm_runtime_share_arenas(self.handle, name.encode(), 1 if create else 0,
                                                  int(stash_bytes)))
        self._w_arena = self._arena(0, np.float32)
        self.k = self._arena(1, np.float32)

    def ipc_export(self) -> bytes:
        buf = (C.c_uint8 * 65536)()
        n = NL.check(self.lib.hm_runtime_ipc_export(self.handle, buf, 65536))
        return bytes(buf[:n])

    def ipc_import(self, blob: bytes) -> None:
        b = (C.c_uint8 * len(blob)).from_buffer_copy(blob)
        NL.check(self.lib.hm_runtime_ipc_import(self.handle, b, len(blob)))

    # -- Harmony-DP communicator -------------------------------------------------
    @staticmethod
    def nccl_path() -> bytes:
        """libnccl.so.2 shipped with torch (the one torch.distributed uses)."""
        import os
        try:
            import nvidia.nccl as nn
            base = list(nn.__path__)[0]
            p = os.path.join(base, "lib", "libnccl.so.2")
            if os.path.exists(p):
                return p.encode()
        except ImportError:
            pass
        return b""

    @classmethod
    def nccl_unique_id(cls) -> bytes:
        buf = (C.c_uint8 * 128)()
        NL.check(NL.lib().hm_nccl_unique_id(cls.nccl_path(), buf))
        return bytes(buf)

    def init_ipc_reduce(self, nranks: int, rank: int) -> None:
        """Harmony-DP with several processes on ONE GPU (tests): the per-pack
        gradient sum runs over CUDA IPC instead of NCCL.  Call before load();
        after it, exchange ipc_export() blobs and ipc_import() every rank's."""
        NL.check(self.lib.hm_runtime_init_ipc_reduce(self.handle, nranks, rank))

    def init_comm(self, unique_id: bytes, nranks: int, rank: int) -> None:
        """Join the job's NCCL communicator (call before load())."""
        buf = (C.c_uint8 * 128).from_buffer_copy(unique_id)
        NL.check(self.lib.hm_runtime_init_comm(self.handle, self.nccl_path(), buf, nranks, rank))

    # -- plan -------------------------------------------------------------------
    def load(self, graph: TaskGraph, machine: MachineModel, profiles: ProfileSet, rank: int = 0) -> None:
        if graph.config is None:
            raise ValidationError("execute needs a scheduler-generated graph")
        if machine.gpu_count != graph.machine.gpu_count:
            raise ValidationError("machine does not match the graph's GPU count")
        dp_update = self.dp_update if graph.mode.value == "dp" else "replicated"
        if self.dp_update == "sharded" and graph.mode.value != "dp":
            raise ValidationError("dp_update='sharded' applies to Harmony-DP graphs")
        plan = NativePlan(graph, machine, profiles, w_fwd_bytes=self.w_fwd_bytes(), dp_update=dp_update)
        if graph.mode.value == "dp":
            samples = gpu_shares(graph.minibatch, machine.gpu_count)[rank]
        else:
            samples = graph.minibatch
        # the native side drops the previous plan first and keeps none on failure
        old, self.plan, self.graph = self.plan, None, None
        rc = self.lib.hm_runtime_load_plan(self.handle, plan.handle, rank, samples)
        if old is not None:
            old.close()
        if rc != 0:
            plan.close()
            NL.check(rc)
        self.plan, self.graph, self.rank, self.samples = plan, graph, rank, samples
        self.machine = machine
        self._checked = None

    def sample_range(self) -> tuple[int, int]:
        """Global sample indices this rank processes."""
        if self.graph is not None and self.graph.mode.value == "dp":
            sh = gpu_shares(self.graph.minibatch, self.machine.gpu_count)
            lo = sum(sh[:self.rank])
            return lo, lo + sh[self.rank]
        return 0, self.samples

    def _gpt_inputs(self, tokens, labels):
        """Validate one minibatch of token ids / labels (shared by step and
        run_steps): both [samples, seq_len], ids in [0, vocab).  Host arrays
        are cast to contiguous int32; CUDA tensors must already be contiguous
        int32 on this runtime's device (an int64 tensor would be read as
        interleaved int32 halves).  Returns (tokens, labels, is_device)."""
        want = (self.samples, self.spec.seq_len)
        V = self.spec.vocab
        if hasattr(tokens, "is_cuda") or hasattr(labels, "is_cuda"):
            import torch
            if not (isinstance(tokens, torch.Tensor) and isinstance(labels, torch.Tensor)
                    and tokens.is_cuda and labels.is_cuda):
                raise ValidationError("tokens and labels must both be host arrays or both CUDA tensors")
            for name, t in (("tokens", tokens), ("labels", labels)):
                if t.dtype != torch.int32:
                    raise ValidationError(f"{name} must be int32 (got {t.dtype})")
                if tuple(t.shape) != want:
                    raise ValidationError(f"{name} must be {list(want)} (got {list(t.shape)})")
                if not t.is_contiguous():
                    raise ValidationError(f"{name} must be contiguous")
                if t.device.index != self.device:
                    raise ValidationError(f"{name} is on cuda:{t.device.index}, the runtime on cuda:{self.device}")
            # the runtime's streams are non-blocking: torch's pending work on
            # the buffers must be finished before they are read
            torch.cuda.current_stream(tokens.device).synchronize()
            key = (tokens.data_ptr(), tokens._version, labels.data_ptr(), labels._version)
            if key != self._checked:  # range check once per buffer version
                lo = min(int(tokens.min()), int(labels.min()))
                hi = max(int(tokens.max()), int(labels.max()))
                if lo < 0 or hi >= V:
                    raise ValidationError(f"token ids / labels must lie in [0, {V}) (got [{lo}, {hi}])")
                self._checked = key
            return tokens, labels, True
        t = np.ascontiguousarray(tokens, dtype=np.int32)
        lb = np.ascontiguousarray(labels, dtype=np.int32)
        for name, a, src in (("tokens", t, tokens), ("labels", lb, labels)):
            if a.shape != want:
                raise ValidationError(f"{name} must be {list(want)} (got {list(a.shape)})")
            if not np.array_equal(a, np.asarray(src)):
                raise ValidationError(f"{name} do not fit int32")
            if a.size and (int(a.min()) < 0 or int(a.max()) >= V):
                raise ValidationError(f"{name} must lie in [0, {V}) (got [{int(a.min())}, {int(a.max())}])")
        return t, lb, False

    @staticmethod
    def _ptr(x) -> int:
        return x.data_ptr() if hasattr(x, "data_ptr") else x.ctypes.data

    def step(self, tokens, labels) -> float:
        """One training iteration on this rank's samples.  ``tokens`` /
        ``labels`` are [samples, seq] int32: numpy (host) or torch CUDA."""
        if self.plan is None:
            raise ValidationError("load() a plan first")
        loss = C.c_double(0.0)
        if self.is_cnn:
            img, lab = self._cnn_inputs(tokens, labels)
            NL.check(self.lib.hm_runtime_run_iteration(self.handle, C.c_void_p(img.data_ptr()),
                                                       C.c_void_p(lab.data_ptr()), int(img.is_cuda), C.byref(loss)))
            return loss.value
        t, lb, dev = self._gpt_inputs(tokens, labels)
        NL.check(self.lib.hm_runtime_run_iteration(self.handle, C.c_void_p(self._ptr(t)), C.c_void_p(self._ptr(lb)),
                                                   int(dev), C.byref(loss)))
        return loss.value

    def _cnn_inputs(self, images, labels):
        """CNN inputs as torch tensors: images [samples, h, w, 64] bf16 (NHWC,
        zero-padded channels), labels [samples] int32; both on one device."""
        import torch
        h, w, c = self.spec.image
        if not isinstance(images, torch.Tensor) or images.dtype != torch.bfloat16 or \
                tuple(images.shape) != (self.samples, h, w, c):
            raise ValidationError(f"images must be a bf16 tensor [{self.samples}, {h}, {w}, {c}]")
        labels = torch.as_tensor(labels, dtype=torch.int32, device=images.device)
        if tuple(labels.shape) != (self.samples,):
            raise ValidationError(f"labels must be [{self.samples}]")
        if labels.numel() and (int(labels.min()) < 0 or int(labels.max()) >= self.spec.classes):
            raise ValidationError(f"labels must lie in [0, {self.spec.classes})")
        images, labels = images.contiguous(), labels.contiguous()
        if images.is_cuda:
            torch.cuda.current_stream(images.device).synchronize()
        return images, labels

    def run_steps(self, n: int, tokens, labels) -> tuple[list[float], float]:
        """``n`` pipelined iterations (cross-iteration overlap); returns the
        per-iteration losses and the device seconds of all n iterations."""
        if self.plan is None:
            raise ValidationError("load() a plan first")
        losses = (C.c_double * n)()
        total = C.c_int64(0)
        if self.is_cnn:
            img, lab = self._cnn_inputs(tokens, labels)
            NL.check(self.lib.hm_runtime_run_steps(self.handle, n, C.c_void_p(img.data_ptr()),
                                                   C.c_void_p(lab.data_ptr()), int(img.is_cuda), losses,
                                                   C.byref(total)))
            return list(losses), total.value / 1e9
        t, lb, dev = self._gpt_inputs(tokens, labels)
        NL.check(self.lib.hm_runtime_run_steps(self.handle, n, C.c_void_p(self._ptr(t)), C.c_void_p(self._ptr(lb)),
                                               int(dev), losses, C.byref(total)))
        return list(losses), total.value / 1e9

    def counters(self) -> dict:
        out = (C.c_int64 * 8)()
        NL.check(self.lib.hm_runtime_counters(self.handle, out, 8))
        return {"kernels": out[0], "iteration_ns": out[1], "device_bytes": out[2],
                "h2d_bytes": out[3], "d2h_bytes": out[4], "p2p_bytes": out[5], "nccl_bytes": out[6],
                "rank_waits": out[7]}

    KERNEL_CLASSES = ("gemm", "attn_fwd", "attn_bwd", "layernorm", "xent", "adam", "other")

    def set_profiling(self, enable: bool) -> None:
        NL.check(self.lib.hm_runtime_set_profiling(self.handle, 1 if enable else 0))

    def kernel_stats(self) -> dict:
        """{class: {ms, flops, bytes, launches}} accumulated while profiling."""
        buf = (C.c_double * 28)()
        NL.check(self.lib.hm_runtime_kernel_stats(self.handle, buf, 28))
        return {c: {"ms": buf[4 * i], "flops": buf[4 * i + 1], "bytes": buf[4 * i + 2],
                    "launches": int(buf[4 * i + 3])} for i, c in enumerate(self.KERNEL_CLASSES)}

    def kernel_launches(self) -> np.ndarray:
        """[n, 5] (class, flops, bytes, event ms, device-clock ms) per launch of
        the last profiled iteration; the device-clock span (first CTA start to
        last CTA end, %globaltimer) is recorded by the GEMM launches, 0 elsewhere."""
        n = self.lib.hm_runtime_kernel_launches(self.handle, None, 0)
        out = np.zeros((max(n, 0), 5), dtype=np.float64)
        if n > 0:
            self.lib.hm_runtime_kernel_launches(self.handle, out.ctypes.data_as(C.POINTER(C.c_double)), n)
        return out

    def gemm_shapes(self) -> list[tuple]:
        """Distinct GEMM calls of the last profiled iteration with their
        counts: [((m, n, k, a_major, b_major, epilogue, has_bias), count)]."""
        n = self.lib.hm_runtime_gemm_shapes(self.handle, None, 0)
        if n <= 0:
            return []
        buf = np.zeros((n, 7), dtype=np.int64)
        self.lib.hm_runtime_gemm_shapes(self.handle, buf.ctypes.data, n)
        out: dict[tuple, int] = {}
        for row in buf:
            key = tuple(int(x) for x in row)
            out[key] = out.get(key, 0) + 1
        return list(out.items())

    def measured_items(self) -> np.ndarray:
        n1 = self.lib.hm_runtime_ledger_count(self.handle)
        n2 = self.lib.hm_runtime_trace_count(self.handle)
        a = np.zeros(n1, dtype=NL.ITEM_DTYPE)
        b = np.zeros(n2, dtype=NL.ITEM_DTYPE)
        if n1:
            NL.check(self.lib.hm_runtime_ledger(self.handle, a.ctypes.data, n1))
        if n2:
            NL.check(self.lib.hm_runtime_trace(self.handle, b.ctypes.data, n2))
        return np.concatenate([b, a])

    def report(self) -> SimReport:
        """SimReport of the last executed iteration (measured CUDA events)."""
        items = self.measured_items()
        c = self.counters()
        return report_from_items(self.graph, self.machine, items, c["iteration_ns"], measured=True)

    def close(self) -> None:
        if getattr(self, "handle", None):
            if self.plan is not None:
                self.plan.close()
            self.lib.hm_runtime_free(self.handle)
            self.handle = None

    def __del__(self) -> None:
        try:
            self.close()
        except Exception:
            pass


def execute(graph: TaskGraph, machine: MachineModel | None = None, profiles: ProfileSet | None = None, *,
            model, batch, steps: int = 1, check_memory: bool = True, rank: int = 0) -> SimReport:
    """Run ``steps`` training iterations of ``graph`` and report the last one.

    ``model`` is a :class:`HarmonyRuntime` (state kept across calls) or a
    :class:`GPTSpec` (a runtime with alpha = ``machine.gpu_mem_capacity`` and
    seed-0 weights is created).  ``batch`` = (tokens, labels), each
    [samples, seq] int32.  Capacity is enforced by the runtime's device pool
    (CapacityViolationError if the plan's buffers exceed alpha)."""
    machine = machine or graph.machine
    if profiles is None:
        raise ValidationError("profiles are required")
    if check_memory:
        from .simulator import check_memory_fit
        check_memory_fit(graph, machine, profiles)
    rt = model
    if isinstance(model, GPTSpec):
        rt = HarmonyRuntime(model, alpha_bytes=machine.gpu_mem_capacity)
        rt.init_weights(0)
    if rt.graph is not graph:
        rt.load(graph, machine, profiles, rank)
    tokens, labels = batch
    losses = [rt.step(tokens, labels) for _ in range(steps)]
    rep = rt.report()
    rep.caveats = rep.caveats + (f"loss={losses[-1]:.6f}",)
    return rep


Runtime = HarmonyRuntime
