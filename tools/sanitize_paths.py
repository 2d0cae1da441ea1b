"""Small runs of every engine path for compute-sanitizer (memcheck / racecheck / synccheck):
tiny MoE layer, GPU Task B, grouped launches over many small experts, the CTA-pair kernel with
several raster groups, in-process P2P expert parallelism (W = 2; W = 4 with sharded shared
experts), both GEMM kernels with
several experts per launch, and the Contiguous Data Mover."""
import os, sys, threading
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np, torch
import synth
from paper_2504_09345_b200 import HostExperts, HostLayer, MoELayer
from gpu_helpers import GpuRun, bf16_tensor

torch.cuda.set_device(0)
# 1. tiny layer + Task B
inp = synth.gen_inputs(synth.CONFIGS["tiny"])
r = GpuRun(inp)
r.run()
tb = synth.gen_taskb(inp.cfg, inp.x)
hl = HostLayer(inp.cfg.hidden, tb.wo, tb.gamma)
a, res = bf16_tensor(tb.attn), bf16_tensor(tb.resid)
o = torch.empty_like(a)
r.layer.taskb_forward(a, res, hl, tb.eps, r.router, r.experts, o)
torch.cuda.synchronize(); r.layer.sync(); hl.close(); r.close()
# 2. many small experts (coalesced DMAs -> grouped GEMM launches), shared experts
cfg = synth.MoEConfig("custom", 21, 256, 256, 32, 4, 300, 2)
inp = synth.gen_inputs(cfg)
r = GpuRun(inp); r.run(); r.run(); r.close()
# 3. CTA-pair kernel with several raster groups per launch
os.environ["MOE_GEMM_PAIR"] = "1"; os.environ["MOE_GEMM_GROUPM"] = "1"
cfg = synth.MoEConfig("custom", 22, 256, 384, 8, 2, 700, 1)
inp = synth.gen_inputs(cfg)
r = GpuRun(inp); r.run(); r.close()
del os.environ["MOE_GEMM_PAIR"], os.environ["MOE_GEMM_GROUPM"]
# 4. in-process P2P expert parallelism, W = 2
W = 2
cfg = synth.MoEConfig("custom", 23, 256, 256, 8, 2, 200, 1)
inp = synth.gen_inputs(cfg)
full = GpuRun(inp)
nl, S, T = cfg.num_experts // W, cfg.num_shared, cfg.tokens
bounds = [T * q // W for q in range(W + 1)]
key = os.urandom(128)
ex, ly, bufs = [], [], []
for q in range(W):
    ids = list(range(q * nl, (q + 1) * nl)) + [cfg.num_experts + s for s in range(S)]
    ex.append(HostExperts(cfg.hidden, cfg.ffn, [inp.w1[i] for i in ids], [inp.w3[i] for i in ids],
                          [inp.w2[i] for i in ids]))
    ly.append(MoELayer(cfg.hidden, cfg.ffn, cfg.num_experts, cfg.top_k, bounds[q + 1] - bounds[q],
                       num_shared=S, world_size=W, rank=q, nccl_unique_id=key, local_ep=True))
    x = bf16_tensor(inp.x[bounds[q]:bounds[q + 1]])
    bufs.append((torch.cuda.Stream(), x, torch.empty_like(x)))
torch.cuda.synchronize()
def work(q):
    s, x, o = bufs[q]
    for _ in range(2):
        ly[q].forward(x, full.router, ex[q], o, stream=s.cuda_stream)
    s.synchronize()
th = [threading.Thread(target=work, args=(q,)) for q in range(W)]
[t.start() for t in th]; [t.join(300) for t in th]
for l in ly: l.close()
for e in ex: e.close()
full.close()
# 4b. sharded shared experts (MOE_FLAG_SHARD_SHARED) over the same transport, W = 4: two ranks
# serve a slice, two serve none
from paper_2504_09345_b200 import shared_slice_weights
W = 4
cfg = synth.MoEConfig("custom", 26, 256, 256, 8, 2, 200, 1)
inp = synth.gen_inputs(cfg)
full = GpuRun(inp)
nl, S, T, ne = cfg.num_experts // W, cfg.num_shared, cfg.tokens, cfg.num_experts
bounds = [T * q // W for q in range(W + 1)]
key = os.urandom(128)
ex, ly, bufs = [], [], []
for q in range(W):
    ids = list(range(q * nl, (q + 1) * nl))
    sl = shared_slice_weights(cfg.ffn, inp.w1[ne:], inp.w3[ne:], inp.w2[ne:], W, q)
    ex.append(HostExperts(cfg.hidden, cfg.ffn, [inp.w1[i] for i in ids], [inp.w3[i] for i in ids],
                          [inp.w2[i] for i in ids], slice_=sl))
    ly.append(MoELayer(cfg.hidden, cfg.ffn, ne, cfg.top_k, max(1, -(-T // W)), num_shared=S,
                       world_size=W, rank=q, nccl_unique_id=key, local_ep=True, shard_shared=True))
    x = bf16_tensor(inp.x[bounds[q]:bounds[q + 1]])
    bufs.append((torch.cuda.Stream(), x, torch.empty_like(x)))
torch.cuda.synchronize()
th = [threading.Thread(target=work, args=(q,)) for q in range(W)]
[t.start() for t in th]; [t.join(300) for t in th]
for l in ly: l.close()
for e in ex: e.close()
full.close()
# 5. both GEMM kernels with several routed experts per launch (MOE_GEMM_ROWS)
cfg = synth.MoEConfig("custom", 24, 768, 1792, 8, 2, 700, 1)
inp = synth.gen_inputs(cfg)
for env in ({"MOE_GEMM_PAIR": "1", "MOE_GEMM_ROWS": "100000"},
            {"MOE_GEMM_PAIR": "0", "MOE_GEMM_ROWS": "100000"}):
    os.environ.update(env)
    r = GpuRun(inp); r.run(); r.close()
    for k in env: del os.environ[k]
# 6. the data mover: small packets, 2 slots, back-to-back calls + Task B
cfg = synth.MoEConfig("custom", 25, 256, 384, 8, 2, 300)
inp = synth.gen_inputs(cfg)
r = GpuRun(inp, mover=True, packet_bytes=64 << 10, num_slots=2)
r.run(); r.run()
tb = synth.gen_taskb(cfg, inp.x)
hl = HostLayer(cfg.hidden, tb.wo, tb.gamma)
a, res = bf16_tensor(tb.attn), bf16_tensor(tb.resid)
o = torch.empty_like(a)
r.layer.taskb_forward(a, res, hl, tb.eps, r.router, r.experts, o)
r.layer.sync(); torch.cuda.synchronize(); hl.close(); r.close()
print("sanitize paths done")
