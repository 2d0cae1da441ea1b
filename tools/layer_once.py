"""Run a few MoE-layer calls at a given token count (for ncu captures)."""
import sys, numpy as np, torch
sys.path.insert(0, ".")
import synth
import paper_2504_09345_b200 as moe
cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "mixtral_8x7b"]
T = int(sys.argv[2]) if len(sys.argv) > 2 and int(sys.argv[2]) > 0 else cfg.tokens
calls = int(sys.argv[3]) if len(sys.argv) > 3 else 2
inp = synth.gen_inputs(cfg, tokens=T)
ex = moe.HostExperts(cfg.hidden, cfg.ffn, inp.w1, inp.w3, inp.w2)
layer = moe.MoELayer(cfg.hidden, cfg.ffn, cfg.num_experts, cfg.top_k, T, num_shared=cfg.num_shared)
x = torch.from_numpy(inp.x.view(np.int16)).view(torch.bfloat16).cuda()
r = torch.from_numpy(inp.router.view(np.int16)).view(torch.bfloat16).cuda()
o = torch.empty_like(x)
for _ in range(calls):
    layer.forward(x, r, ex, o)
torch.cuda.synchronize()
print("done", T)
