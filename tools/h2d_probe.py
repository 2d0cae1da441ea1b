"""Host-link experiments: pinned H2D bandwidth vs transfer size and concurrent streams."""
import sys, time, json
import torch
sys.path.insert(0, ".")
import paper_2504_09345_b200 as moe

res = {"probe_1GB": moe.moe_probe_h2d(0, 1 << 30, 5)}
GB = 1 << 30
h = torch.empty(2 * GB, dtype=torch.uint8).pin_memory()
d = torch.empty(2 * GB, dtype=torch.uint8, device="cuda")
def timed(fn, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize(); t = time.perf_counter(); fn(); torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t)
    return best
for mb in (4, 16, 64, 100, 352, 1024):
    n = mb << 20
    k = (2 * GB) // n
    s = torch.cuda.Stream()
    def f():
        with torch.cuda.stream(s):
            for i in range(k):
                d[i * n:(i + 1) * n].copy_(h[i * n:(i + 1) * n], non_blocking=True)
    t = timed(f)
    res[f"1stream_chunk{mb}MB"] = k * n / t / 1e9
for ns in (2, 4):
    ss = [torch.cuda.Stream() for _ in range(ns)]
    part = (2 * GB) // ns
    def f():
        for j, s in enumerate(ss):
            with torch.cuda.stream(s):
                d[j * part:(j + 1) * part].copy_(h[j * part:(j + 1) * part], non_blocking=True)
    res[f"{ns}streams_concurrent"] = 2 * GB / timed(f) / 1e9
# D2H concurrently with H2D (separate direction)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
h2 = torch.empty(GB, dtype=torch.uint8).pin_memory()
def f():
    with torch.cuda.stream(s1):
        d[:GB].copy_(h[:GB], non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d[GB:2 * GB], non_blocking=True)
res["h2d_plus_d2h_1GB_each_aggregate"] = 2 * GB / timed(f) / 1e9
print(json.dumps(res, indent=1))
