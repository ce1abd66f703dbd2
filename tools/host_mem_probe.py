"""How much pinned host memory can this box hold?  Allocates cudaHostAlloc
chunks of 8 GiB until the target is reached or MemAvailable would drop under a
safety floor, prints MemAvailable after each, frees everything."""
import ctypes, glob, json, os, sys

target_gib = float(sys.argv[1]) if len(sys.argv) > 1 else 176
floor_gib = float(sys.argv[2]) if len(sys.argv) > 2 else 14


def avail_gib():
    for line in open("/proc/meminfo"):
        if line.startswith("MemAvailable:"):
            return int(line.split()[1]) / 2**20
    return 0.0


import torch  # noqa: E402  (loads the CUDA runtime)
torch.cuda.init()
lib = None
for cand in sorted(glob.glob(os.path.join(os.path.dirname(torch.__file__), "lib", "libcudart*.so*"))) + [
        "libcudart.so.12", "/usr/local/cuda/lib64/libcudart.so"]:
    try:
        lib = ctypes.CDLL(cand)
        break
    except OSError:
        continue
out = {"mem_total_gib": None, "start_avail_gib": round(avail_gib(), 1), "steps": []}
for line in open("/proc/meminfo"):
    if line.startswith("MemTotal:"):
        out["mem_total_gib"] = round(int(line.split()[1]) / 2**20, 1)
ptrs, got = [], 0.0
chunk = 8
while got + chunk <= target_gib and avail_gib() - chunk > floor_gib:
    p = ctypes.c_void_p()
    rc = lib.cudaHostAlloc(ctypes.byref(p), ctypes.c_size_t(chunk << 30), 0)
    if rc != 0:
        out["steps"].append({"pinned_gib": got, "error": rc})
        break
    ctypes.memset(p, 0, 1 << 20)
    ptrs.append(p)
    got += chunk
    out["steps"].append({"pinned_gib": got, "avail_gib": round(avail_gib(), 1)})
out["pinned_gib"] = got
for p in ptrs:
    lib.cudaFreeHost(p)
out["end_avail_gib"] = round(avail_gib(), 1)
print(json.dumps(out))
