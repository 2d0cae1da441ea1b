"""Worker of tests/test_gpu_ep_ipc.py: one process = one expert-parallel rank (MOE_FLAG_IPC_EP).

The ranks exchange their CUDA IPC handles through a gloo process group (127.0.0.1), connect,
run `calls` MoE-layer calls on their token slice and return (rank, idx, out bits) through the
queue.  All ranks may share one GPU (the test box has one): CUDA IPC maps same-device memory
across processes like peer memory, so the P2P transport runs unchanged."""
import os
import sys


def run_rank(rank, world, port, cfg_tuple, calls, device, q, shard=False):
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    if root not in sys.path:
        sys.path.insert(0, root)
    try:
        import numpy as np
        import torch
        import torch.distributed as dist

        import synth
        from paper_2504_09345_b200 import HostExperts, MoELayer, shared_slice_weights

        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(device)
        # a BASELINE config by name (its token structure included), or a custom shape tuple
        cfg = synth.CONFIGS[cfg_tuple] if isinstance(cfg_tuple, str) else synth.MoEConfig(*cfg_tuple)
        ne, nl, S, T = cfg.num_experts, cfg.num_experts // world, cfg.num_shared, cfg.tokens
        lo, hi = T * rank // world, T * (rank + 1) // world
        ids = list(range(rank * nl, (rank + 1) * nl)) + [ne + s for s in range(S)]
        inp = synth.gen_inputs(cfg, expert_ids=ids)   # only this rank's experts
        if shard:   # MOE_FLAG_SHARD_SHARED: routed experts + this rank's shared-FFN slice
            sl = shared_slice_weights(cfg.ffn, inp.w1[nl:], inp.w3[nl:], inp.w2[nl:], world, rank)
            experts = HostExperts(cfg.hidden, cfg.ffn, inp.w1[:nl], inp.w3[:nl], inp.w2[:nl],
                                  slice_=sl)
        else:
            experts = HostExperts(cfg.hidden, cfg.ffn, inp.w1, inp.w3, inp.w2)
        cap = max(1, -(-T // world))   # one capacity on every rank (checked at connect)
        layer = MoELayer(cfg.hidden, cfg.ffn, ne, cfg.top_k, cap, num_shared=S,
                         device=device, world_size=world, rank=rank, ipc_ep=True,
                         shard_shared=shard)
        handles = [None] * world
        dist.all_gather_object(handles, layer.ipc_handle())
        layer.ipc_connect(handles)
        layer.ipc_selftest(30.0)
        router = torch.from_numpy(inp.router.view(np.int16)).view(torch.bfloat16).cuda()
        x = torch.from_numpy(np.ascontiguousarray(inp.x[lo:hi]).view(np.int16)).view(torch.bfloat16)
        x = x.reshape(-1, cfg.hidden).cuda()
        out = torch.empty_like(x)
        idx = torch.empty((x.shape[0], cfg.top_k), dtype=torch.int32, device="cuda")
        s = torch.cuda.Stream()
        for _ in range(calls):
            layer.forward(x, router, experts, out, idx, stream=s.cuda_stream)
        s.synchronize()
        layer.sync()
        st = layer.stats()
        q.put((rank, idx.cpu().numpy(), out.view(torch.int16).cpu().numpy(),
               (st["comm_bytes"], st["h2d_weight_bytes"]), None))
        dist.barrier()          # peers may still read this rank's y_recv until they are done
        layer.close()
        experts.close()
        dist.destroy_process_group()
    except Exception as e:  # reported by the parent
        import traceback
        q.put((rank, None, None, None, traceback.format_exc()))
