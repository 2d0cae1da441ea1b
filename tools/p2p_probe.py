"""Ad-hoc LOCAL_EP (in-process P2P) probe: python tools/p2p_probe.py W T NE K S H HI"""
import os, sys, threading
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np, torch
import synth
from paper_2504_09345_b200 import HostExperts, MoELayer
from gpu_helpers import GpuRun, bf16_tensor
W, T, ne, k, S, h, hi = [int(a) for a in sys.argv[1:8]]
cfg = synth.MoEConfig("custom", 16, h, hi, ne, k, T, S)
inp = synth.gen_inputs(cfg)
full = GpuRun(inp); out_full, _, _ = full.run()
nl = ne // W
bounds = [T * r // W for r in range(W + 1)]
key = os.urandom(128)
ex, ly, bufs = [], [], []
for r in range(W):
    ids = list(range(r * nl, (r + 1) * nl)) + [ne + s for s in range(S)]
    ex.append(HostExperts(h, hi, [inp.w1[i] for i in ids], [inp.w3[i] for i in ids], [inp.w2[i] for i in ids]))
for r in range(W):
    ly.append(MoELayer(h, hi, ne, k, max(1, -(-T // W)), num_shared=S, world_size=W, rank=r, nccl_unique_id=key, local_ep=True))
    x = bf16_tensor(inp.x[bounds[r]:bounds[r+1]].reshape(-1, h))
    bufs.append((torch.cuda.Stream(), x, torch.empty_like(x)))
torch.cuda.synchronize()
errs = []
def work(r):
    s, x, o = bufs[r]
    try:
        for _ in range(int(os.environ.get("CALLS", "3"))):
            ly[r].forward(x, full.router, ex[r], o, stream=s.cuda_stream)
        s.synchronize()
    except Exception as e:
        try: ly[r].sync()
        except Exception as e2: errs.append((r, str(e2)[:200]))
        else: errs.append((r, str(e)[:100]))
th = [threading.Thread(target=work, args=(r,)) for r in range(W)]
[t.start() for t in th]; [t.join(120) for t in th]
ok = not errs and all(torch.equal(bufs[r][2], out_full[bounds[r]:bounds[r+1]]) for r in range(W))
print(f"W={W} T={T} ne={ne} k={k} S={S}: {'OK' if ok else 'FAIL'} {errs[:3]}", flush=True)
os._exit(0)
