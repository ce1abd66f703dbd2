"""Micro-benchmarks of the sm_100a kernels (CUDA events, warm-up, L2 flush).

    python tools/kernel_perf.py [gemm|adam|all]
Prints one JSON line per shape with achieved TFLOP/s or GB/s and the fraction
of MEASURED_PEAKS.json.
"""

import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2202_01306_b200 import ops  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d["bf16_tflops"], d["hbm_gbs"], "measured"
    return 1590.0, 6650.0, "fallback"


FLUSH = None
GRAPH = False
SWEEP = None  # list of (bn, cta_pair, splits) to force, None = automatic choice


def flush():
    global FLUSH
    if FLUSH is None:
        FLUSH = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    FLUSH.zero_()


def time_graph(fn, reps=50):
    """Steady-state per-launch time: `reps` back-to-back launches captured in
    one CUDA graph (no flush, no host gaps; consecutive launches overlap
    through programmatic dependent launch where the kernel supports it)."""
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                fn()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def timeit(fn, iters=20, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(iters):
        flush()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    ts.sort()
    return ts[len(ts) // 2]


def bench_gemm():
    tf_peak, _, kind = peaks()
    shapes = [("fwd_qkv", 4096, 4800, 1600, False, False, "bf16"),
              ("fwd_proj", 4096, 1600, 1600, False, False, "resid_f32"),
              ("fwd_head", 4096, 50304, 1600, False, False, "f32"),
              ("dgrad_qkv", 4096, 1600, 4800, False, True, "f32"),
              ("dgrad_fc2", 4096, 6400, 1600, False, True, "dgelu_bf16"),
              ("wgrad_qkv", 4800, 1600, 4096, True, True, "acc_f32"),
              ("wgrad_head", 50304, 1600, 4096, True, True, "acc_f32"),
              ("fwd_fc1", 4096, 6400, 1600, False, False, "gelu_bf16"),
              ("fwd_fc2", 4096, 1600, 6400, False, False, "resid_f32"),
              ("dgrad_fc1", 4096, 1600, 6400, False, True, "f32"),
              ("wgrad_fc1", 6400, 1600, 4096, True, True, "acc_f32"),
              ("fc1_plain_epi", 4096, 6400, 1600, False, False, "bf16"),
              ("fc1_long_k", 4096, 6400, 6400, False, False, "bf16"),
              ("fc1_big_m", 16384, 6400, 1600, False, False, "bf16"),
              ("square8k", 8192, 8192, 8192, False, False, "bf16"),
              ("fwd_40b_qkv", 4096, 24576, 8192, False, False, "bf16")]
    for name, M, N, K, amn, bmn, epi in shapes:
        a = torch.randn(*((K, M) if amn else (M, K)), device="cuda").to(torch.bfloat16)
        b = torch.randn(*((K, N) if bmn else (N, K)), device="cuda").to(torch.bfloat16)
        f32 = epi in ("f32", "acc_f32", "resid_f32")
        d = torch.zeros(M, N, device="cuda", dtype=torch.float32 if f32 else torch.bfloat16)
        bias = torch.zeros(N, device="cuda") if epi not in ("acc_f32", "dgelu_bf16") else None
        aux = None
        if epi == "resid_f32":
            aux = torch.zeros(M, N, device="cuda")
        if epi in ("gelu_bf16", "dgelu_bf16"):
            aux = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16)
        fn = lambda: ops.gemm(a, b, d, a_mn=amn, b_mn=bmn, epi=epi, bias=bias, aux=aux)  # noqa: E731
        ref_ms = None
        if not amn and not bmn:
            rf = lambda: torch.matmul(a, b.t())  # noqa: E731
            ref_ms = time_graph(rf) if GRAPH else timeit(rf)
        for cfg in (SWEEP or [None]):
            if cfg:
                ops.gemm_set_tile(*cfg)
            ms = time_graph(fn) if GRAPH else timeit(fn)
            tf = 2 * M * N * K / ms / 1e9
            tile = ops.gemm_tile(M, N, K, epi, bmn)
            ops.gemm_set_tile(0, 0, 0)
            print(json.dumps({"kernel": "gemm", "timing": "graph50" if GRAPH else "single+flush", "shape": name,
                              "M": M, "N": N, "K": K, "tile": {"bn": tile[0], "cta_pair": tile[1], "splits": tile[2]},
                              "ms": round(ms, 4), "tflops": round(tf, 1), "frac": round(tf / tf_peak, 3),
                              "peak": kind, "cublas_ms": None if ref_ms is None else round(ref_ms, 4)}), flush=True)


def bench_adam():
    _, hbm, kind = peaks()
    n = 256 << 20
    w = torch.zeros(n, device="cuda")
    g = torch.zeros(n, device="cuda")
    k = torch.zeros(2 * n, device="cuda")
    ms = timeit(lambda: ops.adam(w, g, k, lr=1e-4, beta1=0.9, beta2=0.999, eps=1e-8, step=1))
    gbs = 28 * n / ms / 1e6
    print(json.dumps({"kernel": "adam", "params": n, "ms": round(ms, 4), "GBps": round(gbs, 1),
                      "frac": round(gbs / hbm, 3), "peak": kind}), flush=True)


def bench_attn():
    tf_peak, _, kind = peaks()
    for B, S, H, causal in ((4, 1024, 25, True), (8, 512, 16, False), (16, 128, 4, True)):
        DH = 64
        d = H * DH
        qkv = torch.randn(B * S, 3 * d, device="cuda").to(torch.bfloat16)
        out = torch.empty(B * S, d, device="cuda", dtype=torch.bfloat16)
        lse = torch.empty(B * S, H, device="cuda")
        dout = torch.randn(B * S, d, device="cuda").to(torch.bfloat16)
        dqkv = torch.empty_like(qkv)
        fl = 4.0 * B * S * S * H * DH * (0.5 if causal else 1.0)
        ms = timeit(lambda: ops.attn_fwd(qkv, out, lse, batch=B, seq=S, heads=H, head_dim=DH, causal=causal))
        msb = timeit(lambda: ops.attn_bwd(qkv, out, dout, lse, dqkv, batch=B, seq=S, heads=H, head_dim=DH,
                                          causal=causal))
        print(json.dumps({"kernel": "attention", "impl": os.environ.get("HM_ATTN", "tcgen05"), "B": B, "S": S,
                          "H": H, "causal": causal, "fwd_ms": round(ms, 4), "fwd_tflops": round(fl / ms / 1e9, 1),
                          "bwd_ms": round(msb, 4), "bwd_tflops": round(2.5 * fl / msb / 1e9, 1),
                          "peak": tf_peak, "peak_kind": kind}), flush=True)


def bench_attn_sweep():
    """Forward time per 128x128 tile as the tiles per CTA grow (same total
    tiles): separates per-CTA fixed cost from per-tile cost.  Graph-timed,
    back-to-back launches (no flush), so launch latency is excluded."""
    DH = 64
    total_tiles = 2048 * 16
    for causal in (False, True):
        for S in (256, 512, 1024, 2048, 4096):
            nq = S // 128
            per_bh = nq * nq if not causal else nq * (nq + 1) // 2
            BH = max(1, total_tiles // per_bh)
            H = 16
            B = max(1, BH // H)
            d = H * DH
            qkv = torch.randn(B * S, 3 * d, device="cuda").to(torch.bfloat16)
            out = torch.empty(B * S, d, device="cuda", dtype=torch.bfloat16)
            lse = torch.empty(B * S, H, device="cuda")
            ms = time_graph(lambda: ops.attn_fwd(qkv, out, lse, batch=B, seq=S, heads=H, head_dim=DH, causal=causal),
                            reps=10)
            tiles = B * H * per_bh
            fl = 4.0 * B * S * S * H * DH * (0.5 if causal else 1.0)
            print(json.dumps({"kernel": "attn_fwd_sweep", "causal": causal, "S": S, "B": B, "H": H,
                              "ctas": B * H * nq, "tiles": tiles, "ms": round(ms, 4),
                              "ns_per_tile_per_sm": round(ms * 1e6 * 148 / tiles, 1),
                              "tflops": round(fl / ms / 1e9, 1),
                              "env": os.environ.get("HM_ATTN_FWD")}), flush=True)


def bench_ln():
    """LayerNorm fwd / bwd per launch: a CUDA graph of back-to-back launches
    cycling over input sets whose total exceeds L2 (each launch reads cold
    data, launch latency hidden as inside a training step)."""
    _, hbm, kind = peaks()
    for rows, d in ((4096, 1600), (4096, 1024), (8192, 1024), (4096, 8192)):
        nset = max(2, int((400 << 20) // (rows * d * 4 * 3)) + 1)
        sets = []
        for _ in range(nset):
            x = torch.randn(rows, d, device="cuda")
            dy = torch.randn(rows, d, device="cuda")
            sets.append(dict(x=x, dy=dy, y=torch.empty(rows, d, device="cuda", dtype=torch.bfloat16),
                             mu=torch.empty(rows, device="cuda"), rs=torch.empty(rows, device="cuda"),
                             out=torch.empty(rows, d, device="cuda"),
                             ob=torch.empty(rows, d, device="cuda", dtype=torch.bfloat16)))
        g = torch.randn(d, device="cuda")
        b = torch.randn(d, device="cuda")
        dg = torch.zeros(d, device="cuda")
        db = torch.zeros(d, device="cuda")
        it = [0]

        def fwd():
            S = sets[it[0] % nset]
            it[0] += 1
            ops.layernorm_fwd(S["x"], g, b, S["y"], S["mu"], S["rs"])

        def bwd():
            S = sets[it[0] % nset]
            it[0] += 1
            ops.layernorm_bwd(S["dy"], S["x"], S["mu"], S["rs"], g, S["out"], dg, db, resid=S["x"], out_bf16=S["ob"])
        for S in sets:
            ops.layernorm_fwd(S["x"], g, b, S["y"], S["mu"], S["rs"])
        ms = time_graph(fwd, reps=4 * nset)
        msb = time_graph(bwd, reps=4 * nset)
        print(json.dumps({"kernel": "layernorm", "rows": rows, "d": d, "fwd_us": round(ms * 1e3, 2),
                          "fwd_GBps": round(6 * rows * d / ms / 1e6, 1), "bwd_us": round(msb * 1e3, 2),
                          "bwd_GBps": round(18 * rows * d / msb / 1e6, 1), "peak": hbm, "peak_kind": kind,
                          "env": {k: os.environ.get(k) for k in ("HM_LN_FWD", "HM_LN_BWD")}}), flush=True)


def bench_bias():
    """Bias-gradient column sums (graph-timed, input sets larger than L2)."""
    _, hbm, kind = peaks()
    for rows, n, dt in ((4096, 6400, torch.bfloat16), (4096, 1600, torch.float32), (4096, 4800, torch.bfloat16),
                        (200704, 64, torch.bfloat16), (200704, 128, torch.bfloat16), (50176, 256, torch.bfloat16)):
        esz = 2 if dt == torch.bfloat16 else 4
        nset = max(2, int((400 << 20) // (rows * n * esz)) + 1)
        sets = [torch.randn(rows, n, device="cuda").to(dt) for _ in range(nset)]
        db = torch.zeros(n, device="cuda")
        it = [0]

        def fn():
            ops.bias_grad(sets[it[0] % nset], db)
            it[0] += 1
        ms = time_graph(fn, reps=4 * nset)
        print(json.dumps({"kernel": "bias_grad", "rows": rows, "n": n, "dtype": str(dt), "us": round(ms * 1e3, 2),
                          "GBps": round(rows * n * esz / ms / 1e6, 1), "peak": hbm, "peak_kind": kind}), flush=True)


def bench_xent():
    """LM-head cross-entropy (logits fp32 read twice, dlogits bf16 written),
    graph-timed over logits sets larger than L2."""
    _, hbm, kind = peaks()
    for M, V, Vp in ((4096, 50257, 50304), (8192, 30522, 30592)):
        nset = max(2, int((600 << 20) // (M * Vp * 4)) + 1)
        sets = [torch.randn(M, Vp, device="cuda") for _ in range(nset)]
        labels = torch.randint(0, V, (M,), device="cuda", dtype=torch.int32)
        dl = torch.empty(M, Vp, device="cuda", dtype=torch.bfloat16)
        loss = torch.zeros(1, device="cuda", dtype=torch.float64)
        it = [0]

        def fn():
            ops.cross_entropy(sets[it[0] % nset], labels, V, dl, loss, 1.0)
            it[0] += 1
        ms = time_graph(fn, reps=2 * nset)
        print(json.dumps({"kernel": "cross_entropy", "M": M, "V": V, "us": round(ms * 1e3, 1),
                          "GBps_1read": round(M * Vp * 6 / ms / 1e6, 1), "peak": hbm, "peak_kind": kind}), flush=True)


def bench_gemm_bn():
    """Same shapes with the tile width forced (HM_GEMM_BN is read once per
    process, so each width runs in a subprocess)."""
    import subprocess
    for bn in ("128", "256"):
        env = dict(os.environ, HM_GEMM_BN=bn)
        out = subprocess.run([sys.executable, __file__, "gemm"], env=env, capture_output=True, text=True).stdout
        for line in out.splitlines():
            d = json.loads(line)
            d["bn"] = int(bn)
            print(json.dumps(d), flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "gemm_bn":
        bench_gemm_bn()
        sys.exit(0)
    what = sys.argv[1] if len(sys.argv) > 1 else "all"
    if os.environ.get("HM_KP_GRAPH"):
        GRAPH = True
    if what == "gemm_graph":
        GRAPH = True
        what = "gemm"
    if what == "gemm_sweep":
        SWEEP = [(bn, cg, 0) for cg in (1, 2) for bn in (128, 192, 256)]
        what = "gemm"
    if what == "bias":
        bench_bias()
    if what == "xent":
        bench_xent()
    if what == "attn_sweep":
        bench_attn_sweep()
    if what in ("attn", "all"):
        bench_attn()
    if what in ("gemm", "all"):
        bench_gemm()
    if what in ("adam", "all"):
        bench_adam()
    if what in ("ln", "all"):
        bench_ln()
