"""PCIe copy-engine probe: H2D / D2H bandwidth alone and concurrent, with one
or two streams (copy engines) per direction, pinned host memory."""
import json, torch

N = 1 << 30  # 1 GiB per buffer


def run(n_h2d, n_d2h, chunks=8):
    hs = [torch.empty(N, dtype=torch.uint8).pin_memory() for _ in range(max(n_h2d, n_d2h))]
    ds = [torch.empty(N, dtype=torch.uint8, device="cuda") for _ in range(max(n_h2d, n_d2h))]
    hd = [torch.empty(N, dtype=torch.uint8).pin_memory() for _ in range(n_d2h)]
    streams = [torch.cuda.Stream() for _ in range(n_h2d + n_d2h)]
    torch.cuda.synchronize()
    for rep in range(2):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(n_h2d):
            s = streams[i]
            s.wait_event(e0)
            with torch.cuda.stream(s):
                for _ in range(chunks):
                    ds[i].copy_(hs[i], non_blocking=True)
        for j in range(n_d2h):
            s = streams[n_h2d + j]
            s.wait_event(e0)
            with torch.cuda.stream(s):
                for _ in range(chunks):
                    hd[j].copy_(ds[j], non_blocking=True)
        for s in streams:
            e1.wait_stream(s) if hasattr(e1, "wait_stream") else None
            torch.cuda.current_stream().wait_stream(s)
        e1.record()
        torch.cuda.synchronize()
    sec = e0.elapsed_time(e1) / 1e3
    return {"h2d_streams": n_h2d, "d2h_streams": n_d2h, "h2d_gbs": round(n_h2d * chunks * N / sec / 1e9, 1),
            "d2h_gbs": round(n_d2h * chunks * N / sec / 1e9, 1)}


for cfg in ((1, 0), (0, 1), (2, 0), (0, 2), (1, 1), (2, 2), (2, 1), (1, 2)):
    print(json.dumps(run(*cfg)), flush=True)
