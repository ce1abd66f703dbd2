"""Compare the shared-pack activation store after one iteration with a torch
fp32 forward from the same initial weights, tensor by tensor (parity debugging)."""
import json, math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C
import numpy as np
import torch
import torch.nn.functional as F
import paper_2202_01306_b200 as H
from paper_2202_01306_b200 import _native as NL
from paper_2202_01306_b200.model import GPTSpec, gpt_profiles, synthetic_batch
from paper_2202_01306_b200.runtime import HarmonyRuntime

spec = GPTSpec(int(os.environ.get("NL", 2)), int(os.environ.get("DM", 2048)), int(os.environ.get("NH", 16)), 256, 1024)
u, D = int(os.environ.get("U", 1)), int(os.environ.get("DD", 2))
packs = ((0, spec.n_layer - 1),)
cfg = H.Configuration(u, packs, u, packs, D, H.Mode.PP)
prof = gpt_profiles(spec)
mach = H.MachineModel(gpu_count=1, gpu_mem_capacity=48 << 30, pcie_bandwidth=55_000_000_000)
g = H.generate_task_graph(cfg, mach, prof)
rt = HarmonyRuntime(spec, alpha_bytes=48 << 30)
rt.init_weights(0)
w0 = torch.from_numpy(rt.w.copy()).cuda()
rt.load(g, mach, prof)
tok, lab = synthetic_batch(spec, D)
loss = rt.step(tok, lab)
S, d, Hh, Vp = spec.seq_len, spec.d_model, spec.n_head, spec.vocab_padded
names = ["x", "mean1", "rstd1", "lse", "h1", "mean2", "rstd2", "ln1", "qkv", "o", "ln2", "hpre", "a"]
sizes = [S * d * 4, S * 4, S * 4, S * Hh * 4, S * d * 4, S * 4, S * 4, S * d * 2, S * 3 * d * 2, S * d * 2, S * d * 2,
         S * 4 * d * 2, S * 4 * d * 2]
def al(x): return (x + 255) // 256 * 256
def read(off, nbytes, dtype):
    buf = np.zeros(nbytes // np.dtype(dtype).itemsize, dtype=dtype)
    NL.check(rt.lib.hm_runtime_debug_read(rt.handle, 0, off, nbytes, buf.ctypes.data))
    return buf
def bf16(raw):  # uint16 -> float32
    return torch.from_numpy((raw.astype(np.uint32) << 16).view(np.float32)).cuda()
def views(L):
    out, o = {}, int(rt.w_off[L])
    shapes = {"wte": (Vp, d), "wpe": (S, d), "w_qkv": (3 * d, d), "w_proj": (d, d), "w_fc1": (4 * d, d),
              "w_fc2": (d, 4 * d), "w_head": (Vp, d)}
    for name, n in spec.layer_segments(L):
        t = w0[o:o + n]
        out[name] = t.view(*shapes[name]) if name in shapes else t
        o += n
    return out
tk = torch.from_numpy(tok).long().cuda()
x = None
base = 0
res = {"loss": loss}
for L in range(spec.n_layer):
    p = views(L)
    if L == 0:
        x = p["wte"][tk] + p["wpe"][None]
    ref = {}
    ref["x"] = x
    ln1 = F.layer_norm(x, (d,), p["ln1_g"], p["ln1_b"], 1e-5); ref["ln1"] = ln1
    qkv = ln1 @ p["w_qkv"].t() + p["b_qkv"]; ref["qkv"] = qkv
    q, k, v = qkv.view(D, S, 3, Hh, d // Hh).permute(2, 0, 3, 1, 4)
    sc = (q @ k.transpose(-1, -2)) / math.sqrt(d // Hh)
    sc = sc.masked_fill(torch.triu(torch.ones(S, S, device="cuda", dtype=torch.bool), 1), float("-inf"))
    o = (torch.softmax(sc, -1) @ v).permute(0, 2, 1, 3).reshape(D, S, d); ref["o"] = o
    h1 = x + o @ p["w_proj"].t() + p["b_proj"]; ref["h1"] = h1
    ln2 = F.layer_norm(h1, (d,), p["ln2_g"], p["ln2_b"], 1e-5); ref["ln2"] = ln2
    hpre = ln2 @ p["w_fc1"].t() + p["b_fc1"]; ref["hpre"] = hpre
    a = F.gelu(hpre, approximate="tanh"); ref["a"] = a
    y = h1 + a @ p["w_fc2"].t() + p["b_fc2"]
    head = L == spec.n_layer - 1
    off = base
    for nm, sz in zip(names, sizes):
        if nm in ref:
            raw = read(off, D * sz, np.float32 if sz in (S * d * 4,) and nm in ("x", "h1") else np.uint16)
            got = torch.from_numpy(raw).cuda() if raw.dtype == np.float32 else bf16(raw)
            r = ref[nm].reshape(-1).float()
            res[f"L{L}.{nm}"] = round(((got - r).norm() / r.norm()).item(), 6)
        off += al(D * sz)
    if head:
        off += al(D * S * d * 4) + 2 * al(D * S * 4) + al(D * S * d * 2) + al(D * S * Vp * 2)
    base = off
    x = y
print(json.dumps(res))
