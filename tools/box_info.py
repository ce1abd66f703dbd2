"""Host/GPU facts of the GPU box: cores, RAM, PCIe H2D/D2H GB/s (pinned)."""
import json, os, time
import torch
def bw(direction, nbytes=1 << 30, iters=5):
    h = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    for _ in range(2):
        (d.copy_(h, non_blocking=True) if direction == "h2d" else h.copy_(d, non_blocking=True))
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        (d.copy_(h, non_blocking=True) if direction == "h2d" else h.copy_(d, non_blocking=True))
    e.record(); torch.cuda.synchronize()
    return nbytes * iters / (s.elapsed_time(e) / 1e3) / 1e9
mem = os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES") / 2**30
out = {"cores": len(os.sched_getaffinity(0)), "ram_gib": round(mem, 1), "gpu": torch.cuda.get_device_name(0),
       "h2d_gbs": round(bw("h2d"), 2), "d2h_gbs": round(bw("d2h"), 2)}
print(json.dumps(out))
