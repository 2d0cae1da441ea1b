#!/usr/bin/env python
"""Benchmark of the streamed-weight MoE layer (BASELINE.json metric: "Mixtral-8x7B MoE-layer
tokens/s, weights streamed from host; % of roofline").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config mixtral_8x7b] [--impl ours|reference]

A step = one full MoE-layer call (router GEMM + top-k gating, permute, grouped SwiGLU expert
GEMMs, combine) with ALL of the layer's expert weights streamed from pinned host DRAM during the
step; consecutive steps cycle L=2 distinct layers (distinct host weight sets), and staging holds
fewer expert slots than the layer has experts (2 at C1; asserted), so nothing is reused across
steps.  The 2.8 GB of weights streamed per step are far larger than L2 (126 MB), which is the
"inputs larger than L2" rule.  --taskb times GPU Task B (O-projection + RMSNorm + MoE); N > 1
runs under torchrun with expert parallelism (P2P transport over CUDA IPC, NCCL fallback).

Printed JSON (one line, rank 0): value = tokens/s over the timed region (device CUDA events on the
launching stream, max over ranks), plus `roofline` (dominant kernel: the GEMM1+SwiGLU tcgen05
kernel vs measured bf16 peak), `roofline_step` (the north-star roofline: max(expert FLOPs /
tensor peak, streamed bytes / measured host link)), `e2e` (same metric through the host-buffer C
ABI entry point), `cpu_baseline` (the oracle on a bounded token sample), `clocks`, `gpu_launches`.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Mixtral-8x7B MoE-layer tokens/s, weights streamed from host; % of roofline"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)   # >= 20 timed calls
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="mixtral_8x7b")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--layers", type=int, default=2)
    ap.add_argument("--tokens", type=int, default=0,
                    help="override the config's token count (e.g. 131072 = 2 x n_real at C1: the "
                         "compute-bound regime of the paper's profiler, PAPER.md:608-615)")
    ap.add_argument("--packet-mb", type=float, default=0.0)
    ap.add_argument("--mover", action="store_true",
                    help="expert copies through the library's data-mover thread (MOE_FLAG_MOVER)")
    ap.add_argument("--slots", type=int, default=0, help="expert staging slots (0 = auto)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--cpu-one-thread-tokens", type=int, default=8,
                    help="tokens of the one-thread oracle sample (SURVEY §8(d): 64 = all of C0, "
                         "256 = a C1 slice)")
    ap.add_argument("--taskb", action="store_true",
                    help="time GPU Task B (O-projection + RMSNorm + MoE layer, streamed Wo) "
                         "instead of the MoE layer alone (no cpu leg)")
    ap.add_argument("--partitions", type=int, default=1, choices=[1, 2],
                    help="--taskb e2e: 2 = VSLPipe's alpha / beta token partitions through one "
                         "stream of the layer's weights (moe_taskb_forward2_host, PAPER.md:795-801)")
    ap.add_argument("--shared", default="auto", choices=["auto", "replicated", "sharded"],
                    help="shared experts under EP: sharded by intermediate columns across the "
                         "ranks (MOE_FLAG_SHARD_SHARED, P2P transport) or replicated on every "
                         "rank; auto = sharded when N > 1 with the p2p transport")
    ap.add_argument("--ep-transport", default="p2p", choices=["p2p", "nccl"],
                    help="N > 1: p2p = fused dispatch/combine over peer memory (CUDA IPC), "
                         "falling back to NCCL if the peers cannot be mapped; nccl = NCCL "
                         "all-to-all")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def spread_devices(world: int):
    """The W GPUs a run uses when it has fewer ranks than the box has GPUs (spread
    W = 2 / 4 over PCIe switches and sockets, so ranks do not share a host uplink): greedy --
    GPU 0 first, then repeatedly the GPU whose closest already-chosen GPU is topologically
    farthest (NVML common-ancestor level: system > NUMA node > host bridge > PCIe switches), ties
    to the lowest index.  Deterministic, so every rank computes the same list.  Identity when
    every visible GPU is used, NVML is missing, or MOE_BENCH_SPREAD=0."""
    import torch
    n = torch.cuda.device_count()
    if world >= n or os.environ.get("MOE_BENCH_SPREAD") == "0":
        return list(range(world)), "identity"
    try:
        import pynvml
        pynvml.nvmlInit()
        hs = []
        for d in range(n):
            p = torch.cuda.get_device_properties(d)
            busid = f"{p.pci_domain_id:08x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
            hs.append(pynvml.nvmlDeviceGetHandleByPciBusId(busid))
        chosen = [0]
        while len(chosen) < world:
            best, best_lvl = None, -1
            for d in range(n):
                if d in chosen:
                    continue
                lvl = min(pynvml.nvmlDeviceGetTopologyCommonAncestor(hs[d], hs[c]) for c in chosen)
                if lvl > best_lvl:
                    best, best_lvl = d, lvl
            chosen.append(best)
        return sorted(chosen), "nvml topology spread"
    except Exception as e:  # noqa: BLE001 -- fall back to a stride over the visible GPUs
        return [r * (n // world) for r in range(world)], f"stride ({str(e)[:60]})"


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return {"hbm_gbs": d.get("hbm_gbs", 6650.0), "bf16_tflops": d.get("bf16_tflops", 1590.0),
                "bf16_tflops_sustained": d.get("bf16_tflops_sustained", 1400.0),
                "source": "measured (MEASURED_PEAKS.json)"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
            "source": "fallback (B200_PROFILING.md)"}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={self.device}",
                                       f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                       "-lms", "200"], stdout=self.f, stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        self.p.terminate()
        try:
            self.p.wait(5)
        except subprocess.TimeoutExpired:
            self.p.kill()
        self.f.flush()
        rows = [l.split(",") for l in open(self.f.name).read().strip().splitlines() if l.strip()]
        os.unlink(self.f.name)
        sm, smax, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                sm.append(float(r[1]))
                smax = max(smax, float(r[2]))
                for n, v in zip(names, r[5:9]):
                    if v.strip() == "Active":
                        reasons.add(n)
            except (ValueError, IndexError):
                continue
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------------------------
def cpu_baseline(inp, seconds: float, one_thread_tokens: int = 8) -> dict:
    """The oracle as it stands, on a bounded token sample of the same workload (rank 0 only)."""
    import oracle
    cfg = inp.cfg
    cores = oracle.num_threads()
    n = max(8, cores)
    done, elapsed, rounds = 0, 0.0, 0
    while elapsed < seconds and done < cfg.tokens:
        lo = done % inp.x.shape[0]
        xs = inp.x[lo:lo + n]
        t0 = time.perf_counter()
        oracle.forward(xs, inp.router, inp.w1, inp.w3, inp.w2, cfg.top_k, cfg.num_shared)
        elapsed += time.perf_counter() - t0
        done += xs.shape[0]
        rounds += 1
        if elapsed < seconds / 8:
            n *= 2
    # one host thread on a small sample: the scaling of the oracle itself
    one = None
    try:
        oracle.set_num_threads(1)
        n1 = min(max(1, one_thread_tokens), inp.x.shape[0])
        t0 = time.perf_counter()
        oracle.forward(inp.x[:n1], inp.router, inp.w1, inp.w3, inp.w2, cfg.top_k, cfg.num_shared)
        dt = time.perf_counter() - t0
        one = {"value": n1 / dt, "unit": "tokens/s", "cores": 1,
               "sample": f"{n1} tokens of the {cfg.name} layer, 1 OpenMP thread ({dt:.2f} s)",
               "extrapolated_full_layer_s": cfg.tokens * dt / n1,
               "extrapolated_note": f"all {cfg.tokens} tokens at the sample's rate (extrapolated)"}
    finally:
        oracle.set_num_threads(cores)
    return {"value": done / elapsed, "unit": "tokens/s", "cores": cores, "kind": "oracle",
            "sample": f"{done} of {cfg.tokens} tokens of the {cfg.name} layer ({rounds} calls, "
                      f"{elapsed:.1f} s, fp64 router + fp32 experts, OpenMP)",
            "one_thread": one, "host": host_cpu_info()}


def host_cpu_info() -> dict:
    """lscpu model / sockets / cores / SMT of the box the oracle ran on."""
    info = {}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        keys = {"Model name": "model", "Socket(s)": "sockets", "Core(s) per socket":
                "cores_per_socket", "Thread(s) per core": "threads_per_core",
                "NUMA node(s)": "numa_nodes"}
        for line in out.splitlines():
            k, _, v = line.partition(":")
            if k.strip() in keys:
                info[keys[k.strip()]] = v.strip()
    except Exception as e:  # noqa: BLE001 -- informational only
        info["error"] = str(e)[:80]
    return info


def run_reference(args):
    """--impl reference: the CPU oracle timed on the host cores (rank 0 only)."""
    import oracle
    import synth
    rank, world, _ = dist_env()
    if rank != 0:
        return
    cfg = synth.CONFIGS[args.config]
    oracle.build()
    inp = synth.gen_inputs(cfg)
    cores = oracle.num_threads()
    n = max(8, cores)
    for i in range(args.warmup):
        oracle.forward(inp.x[:n], inp.router, inp.w1, inp.w3, inp.w2, cfg.top_k, cfg.num_shared)
    times = []
    for i in range(args.steps):
        lo = (i * n) % (cfg.tokens - n + 1)
        t0 = time.perf_counter()
        oracle.forward(inp.x[lo:lo + n], inp.router, inp.w1, inp.w3, inp.w2, cfg.top_k,
                       cfg.num_shared)
        times.append(time.perf_counter() - t0)
    tot = sum(times)
    value = n * args.steps / tot
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * tot / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": cfg.name, "tokens": cfg.tokens, "hidden": cfg.hidden,
                       "ffn": cfg.ffn, "experts": cfg.num_experts, "top_k": cfg.top_k,
                       "tokens_per_step": n},
            "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": cores, "kind": "oracle",
                             "sample": f"{n} tokens per step of the {cfg.name} layer",
                             "host": host_cpu_info()},
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------------------------
def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import synth
    import paper_2504_09345_b200 as moe
    from paper_2504_09345_b200 import build as moe_build
    from paper_2504_09345_b200 import ledger

    rank, world, local = dist_env()
    # MOE_BENCH_SHARE_GPU=1 (path check only, timings meaningless): every rank on GPU 0 and a
    # gloo group for the bench's own plumbing -- exercises the N > 1 code path on a 1-GPU box
    # with the P2P transport (NCCL refuses two ranks on one GPU).
    share = os.environ.get("MOE_BENCH_SHARE_GPU") == "1"
    placement = "shared GPU 0 (path check)" if share else "identity"
    if share:
        local = 0
    elif world > 1 and int(os.environ.get("LOCAL_WORLD_SIZE", world)) == world:
        devs, placement = spread_devices(world)   # single node: spread the ranks' GPUs
        local = devs[local]
    torch.cuda.set_device(local)
    if world > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    if rank == 0:
        moe_build.build()
    if world > 1:
        dist.barrier()
    peaks = load_peaks()
    cfg = synth.CONFIGS[args.config]
    if args.tokens:
        cfg = cfg.with_tokens(args.tokens)
    T = cfg.tokens                      # global tokens per step (strong scaling over ranks)
    if T % world or cfg.num_experts % world:
        raise SystemExit(f"{cfg.name}: tokens/experts do not split over {world} ranks")
    Tr = T // world
    nl = cfg.num_experts // world
    ids = list(range(rank * nl, (rank + 1) * nl)) + [cfg.num_experts + s for s in range(cfg.num_shared)]
    shard = (cfg.num_shared > 0 and world > 1 and
             (args.shared == "sharded" or (args.shared == "auto" and args.ep_transport == "p2p")))
    if shard and args.ep_transport != "p2p":
        raise SystemExit("--shared sharded needs the p2p transport")

    def allmax(v):
        if world == 1:
            return v
        t = torch.tensor([float(v)], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def allsum(v):
        if world == 1:
            return v
        t = torch.tensor([float(v)], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    # ---- pin this rank's host threads (and so its pinned weight pages, first-touched by
    # cudaHostAlloc) to the CPUs local to its GPU, so each GPU streams from its own NUMA node
    # (the paper used numactl).  MOE_BENCH_NO_AFFINITY=1 disables it.
    all_cpus = os.sched_getaffinity(0)
    affinity = {"numa_local": False, "cpus": len(all_cpus)}
    if os.environ.get("MOE_BENCH_NO_AFFINITY") != "1":
        try:
            import pynvml
            pynvml.nvmlInit()
            p = torch.cuda.get_device_properties(local)
            busid = f"{p.pci_domain_id:08x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
            pynvml.nvmlDeviceSetCpuAffinity(pynvml.nvmlDeviceGetHandleByPciBusId(busid))
            affinity = {"numa_local": True, "cpus": len(os.sched_getaffinity(0)),
                        "gpu_pci": busid}
        except Exception as e:  # noqa: BLE001 -- affinity is an optimisation; report and go on
            affinity["error"] = str(e)[:120]

    # ---- inputs: L layers; this rank's token slice and only its own experts (pinned, packed)
    layers = [synth.gen_inputs(cfg, layer=l, expert_ids=ids) for l in range(args.layers)]
    if shard:   # routed experts + this rank's column slice of the concatenated shared FFN
        experts = [moe.HostExperts(cfg.hidden, cfg.ffn, l.w1[:nl], l.w3[:nl], l.w2[:nl],
                                   slice_=moe.shared_slice_weights(cfg.ffn, l.w1[nl:], l.w3[nl:],
                                                                   l.w2[nl:], world, rank))
                   for l in layers]
    else:
        experts = [moe.HostExperts(cfg.hidden, cfg.ffn, l.w1, l.w3, l.w2) for l in layers]
    xslice = [np.ascontiguousarray(l.x[rank * Tr:(rank + 1) * Tr]) for l in layers]
    xs = [torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).cuda() for x in xslice]
    routers = [torch.from_numpy(l.router.view(np.int16)).view(torch.bfloat16).cuda() for l in layers]
    outs = [torch.empty_like(x) for x in xs]
    idxs = [torch.empty((Tr, cfg.top_k), dtype=torch.int32, device="cuda") for _ in layers]
    gws = [torch.empty((Tr, cfg.top_k), dtype=torch.float32, device="cuda") for _ in layers]

    if world > 1:
        dist.barrier()   # all ranks probe their host links at the same time (shared host DRAM)
    probe_gbs = moe.moe_probe_h2d(local, 1 << 30, 5)   # paper's method: 1 GB pinned H2D copies
    transport0 = "single" if world == 1 else args.ep_transport

    def make_layer(profile):
        """This rank's context: the P2P transport over CUDA IPC when asked and every rank can map
        its peers (checked by a self-test), else NCCL.  Returns (layer, transport)."""
        transport, layer, uid = transport0, None, None
        mk = dict(num_shared=cfg.num_shared, device=local, profile=profile,
                  packet_bytes=int(args.packet_mb * 2 ** 20), mover=args.mover, world_size=world,
                  rank=rank, num_slots=args.slots, shard_shared=shard)
        if transport == "p2p":   # CUDA IPC peer mapping; every rank must succeed, else NCCL
            # Every rank reaches the same collectives whatever fails locally (a rank that cannot
            # build its context still joins the handle exchange with None), so a local failure
            # never leaves the others waiting in a collective it skipped.
            err, hnd = None, None
            try:
                layer = moe.MoELayer(cfg.hidden, cfg.ffn, cfg.num_experts, cfg.top_k, Tr,
                                     ipc_ep=True, **mk)
                hnd = layer.ipc_handle()
            except Exception as e:  # noqa: BLE001 -- reported below, then the NCCL transport
                err = e
            handles = [None] * world
            dist.all_gather_object(handles, hnd)
            ok = 0.0
            if err is None and all(x is not None for x in handles):
                try:
                    layer.ipc_connect(handles)
                    layer.ipc_selftest(5.0)   # flags + rows through the mapping (peers time out
                    ok = 1.0                  # instead of hanging if one rank could not connect)
                except Exception as e:  # noqa: BLE001
                    err = e
            elif err is None:
                err = RuntimeError("a peer could not build its IPC context")
            if err is not None:
                print(f"[bench] rank {rank}: P2P transport unavailable ({err}); using NCCL",
                      file=sys.stderr, flush=True)
            if allmax(1.0 - ok) > 0:
                if layer is not None:
                    layer.close()
                if shard:
                    raise SystemExit("P2P transport unavailable: sharded shared experts need it "
                                     "(run with --shared replicated)")
                layer, transport = None, "nccl"
        if world > 1 and transport == "nccl":
            obj = [moe.moe_nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            uid = obj[0]
        if layer is None:
            layer = moe.MoELayer(cfg.hidden, cfg.ffn, cfg.num_experts, cfg.top_k, Tr,
                                 nccl_unique_id=uid, **mk)
        return layer, transport

    def drop_layer(layer):
        layer.sync()
        if world > 1:
            dist.barrier()   # P2P: peers may read this rank's buffers until their combine ends
        layer.close()

    stream = torch.cuda.Stream()
    sh = stream.cuda_stream
    layer_bytes = 0
    if args.taskb:   # GPU Task B: per layer a streamed Wo + gamma blob, attention output, residual
        args.no_cpu = True
        tbs = [synth.gen_taskb(cfg, l.x, layer=i) for i, l in enumerate(layers)]
        hls = [moe.HostLayer(cfg.hidden, tb.wo, tb.gamma) for tb in tbs]
        layer_bytes = hls[0].nbytes

        def _dev(bits):
            return torch.from_numpy(np.ascontiguousarray(bits[rank * Tr:(rank + 1) * Tr]).view(np.int16)).view(torch.bfloat16).cuda()
        attns = [_dev(tb.attn) for tb in tbs]
        resids = [_dev(tb.resid) for tb in tbs]

    def step(i):
        l = i % args.layers
        if args.taskb:
            layer.taskb_forward(attns[l], resids[l], hls[l], tbs[l].eps, routers[l], experts[l],
                                outs[l], idxs[l], gws[l], stream=sh)
            return
        layer.forward(xs[l], routers[l], experts[l], outs[l], idxs[l], gws[l], stream=sh)

    # e2e inputs: host token buffers through the host-buffer entry points (H2D tokens + D2H out)
    if not args.no_e2e:
        xh = [torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).pin_memory() for x in xslice]
        oh = [torch.empty_like(x).pin_memory() for x in xh]
        if args.taskb:   # attention output from host memory (the paper's CPU attention)
            xh = [a.cpu().pin_memory() for a in attns]
        half = Tr // 2   # --partitions 2: alpha = the first half of the rank's tokens
        if args.partitions == 2:
            if not args.taskb:
                raise SystemExit("--partitions 2 needs --taskb (VSLPipe's partitions are Task B's)")
            xh2 = [[x[:half], x[half:]] for x in xh]
            oh2 = [[o[:half], o[half:]] for o in oh]
            rs2 = [[r[:half], r[half:]] for r in resids]

    def step_h(i):
        l = i % args.layers
        if args.taskb and args.partitions == 2:
            layer.taskb_forward2_host(xh2[l], rs2[l], hls[l], tbs[l].eps, routers[l],
                                      experts[l], oh2[l], stream=sh)
            return
        if args.taskb:
            layer.taskb_forward_host(xh[l], resids[l], hls[l], tbs[l].eps, routers[l],
                                     experts[l], oh[l], stream=sh)
            return
        layer.forward_host(xh[l], routers[l], experts[l], oh[l], stream=sh)

    def timed(fn, sampler=None, fence=None):
        for i in range(args.warmup):
            fn(i)
        torch.cuda.synchronize()
        layer.reset_stats()          # per-kernel stats cover the timed steps only
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
        if sampler is not None:
            sampler.start()
        evs[0].record(stream)
        for i in range(args.steps):
            fn(args.warmup + i)
            if fence is not None and i == args.steps - 1:
                fence()          # the last step's result copy (library D2H stream) is in the region
            evs[i + 1].record(stream)
        torch.cuda.synchronize()
        if sampler is not None:
            sampler.result = sampler.stop()
        if world > 1:
            dist.barrier()
        per_step = sorted(evs[i].elapsed_time(evs[i + 1]) for i in range(args.steps))
        q = lambda f: per_step[min(len(per_step) - 1, int(f * len(per_step)))]  # noqa: E731
        timed.dist = {"p10": q(0.1), "p50": q(0.5), "p90": q(0.9)}
        return allmax(evs[0].elapsed_time(evs[-1])) / args.steps

    # ---- pass 1 (the headline): the library's default configuration, MOE_FLAG_PROFILE off --
    # no event brackets or clock probes in the timed region
    layer, transport = make_layer(False)
    comm_nranks = layer.group_size()
    if world > 1:
        print(f"[bench] rank {rank}: expert-parallel transport {transport}, group size "
              f"{comm_nranks} (NCCL: ncclCommCount)", file=sys.stderr, flush=True)
    clocks = ClockSampler(local)
    ms = timed(step, clocks)
    step_dist = dict(timed.dist)
    clk = clocks.result
    value = T / (ms / 1e3)
    ems = None
    if not args.no_e2e:
        ems = timed(step_h, fence=lambda: layer.wait_output(sh))
        last = (args.warmup + args.steps - 1) % args.layers
        e2e_match = bool(allmax(0.0 if torch.equal(oh[last].cuda(), outs[last]) else 1.0) == 0.0)
    # single-call latency: one isolated call (no cross-call prefetch), all ranks together
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    l0, l1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0.record(stream)
    step(args.warmup + args.steps)
    l1.record(stream)
    torch.cuda.synchronize()
    latency_ms = allmax(l0.elapsed_time(l1))
    drop_layer(layer)
    # the link probe again, after the headline pass: a shared host's other traffic makes single
    # probes vary by ~10% from box to box; the roofline takes the better of the two (the
    # bandwidth the link demonstrably has), both are reported
    if world > 1:
        dist.barrier()
    probe_after = moe.moe_probe_h2d(local, 1 << 30, 5)
    probe_before, probe_gbs = probe_gbs, max(probe_gbs, probe_after)

    # ---- pass 2 (the explanation): MOE_FLAG_PROFILE on -- per-kernel CUDA-event times, the
    # dominant kernel's roofline, the in-kernel SM clock, copy-stream busy time
    layer, _ = make_layer(True)
    ms_prof = timed(step)
    st = layer.stats()
    est = None
    if not args.no_e2e:
        timed(step_h, fence=lambda: layer.wait_output(sh))
        est = layer.stats()
    # every expert is re-streamed every call: fewer staging slots than experts per call (the
    # library enforces it for explicit slot counts; asserted here for the run's auto choice)
    streamed = nl + (int(experts[0].slice_bytes > 0) if shard else cfg.num_shared)
    assert st["num_slots"] == 2 or st["num_slots"] < streamed, st["num_slots"]
    assert st["h2d_weight_bytes"] >= args.steps * experts[0].nbytes, \
        "weights were not re-streamed every step"

    # ---- work ledger (experts hit: from the routing of the timed layers, all ranks)
    cnt = torch.zeros(cfg.num_experts, dtype=torch.int64, device="cuda")
    for l in range(args.layers):
        cnt += torch.bincount(idxs[l].flatten().long(), minlength=cfg.num_experts)
    if world > 1:
        dist.all_reduce(cnt)
    hit = int((cnt > 0).sum().item())
    work = ledger.layer_work(T, cfg.hidden, cfg.ffn, cfg.num_experts, cfg.top_k, cfg.num_shared,
                             experts_hit=hit)
    rank_bytes = experts[0].nbytes + layer_bytes
    step_weight_bytes = work.weight_bytes + world * layer_bytes
    oproj_flops = 2.0 * T * cfg.hidden * cfg.hidden if args.taskb else 0.0
    # Host-link roofline on ALGORITHMIC bytes: the layer's weights once, split over W links
    # -- shared experts (and Task B's Wo) replicated on every rank are charged
    # against us, not credited.  The slowest rank's probe is the link bandwidth.
    alg_rank_bytes = (work.weight_bytes + layer_bytes) / world
    t_io = alg_rank_bytes / (-allmax(-probe_gbs) * 1e9)
    t_tc = (work.expert_flops + oproj_flops) / world / (peaks["bf16_tflops_sustained"] * 1e12)
    t_roof = max(t_io, t_tc)
    # dominant kernel: GEMM1 (+SwiGLU).  FLOPs per launch over all ranks / avg launch time.
    g1_ms, g1_n = allsum(st["gemm1_ms"]), allsum(st["gemm1_launches"])
    g1_flops_total = work.gemm1_flops * args.steps
    g1_flops_launch = g1_flops_total / max(1.0, g1_n)
    g1_launch_ms = g1_ms / max(1.0, g1_n)
    achieved_tf = g1_flops_launch / (g1_launch_ms * 1e-3) / 1e12 if g1_launch_ms > 0 else 0.0
    # DRAM bytes per GEMM1 launch from one `ncu --set full` capture (dram__bytes_read.sum +
    # dram__bytes_write.sum) of the committed build, kept in profiles/ncu_traffic.json with its
    # provenance (round, capture command) -- ncu cannot run inside the timed bench
    traffic, traffic_src = None, None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        tj = json.load(open(tp))
        key = cfg.name + ("@%d" % T if args.tokens else "")
        traffic = tj.get(key, {}).get("gemm1_dram_bytes_per_launch")
        traffic_src = tj.get(key, {}).get("source", tj.get("source")) if traffic else None
    # Peak: the BURST cuBLAS figure.  The kernel runs inside a long step, but the step is
    # host-link bound and the GPU idles between expert GEMMs (~0.2-ms bursts, nvidia-smi sees
    # boost clock, `clocks`), so the burst peak is the conservative denominator; the sustained-peak
    # fraction is reported beside it, and so is the SM clock measured INSIDE the kernel (power
    # management still lowers it during the burst: ~1.5 GHz, `sm_mhz_in_kernel`).
    roofline = {"kernel": "expert GEMM1 + fused SwiGLU (a5): tcgen05 expert_gemm_pair_kernel / "
                          "expert_gemm_kernel<256,0>, chosen per launch by the wave model",
                "bound": "tensor",
                "achieved": achieved_tf, "peak": peaks["bf16_tflops"],
                "unit": "TFLOP/s", "frac": achieved_tf / peaks["bf16_tflops"],
                "frac_of_sustained_peak": achieved_tf / peaks["bf16_tflops_sustained"],
                "traffic": traffic if world == 1 else None,
                "traffic_source": traffic_src if world == 1 else None,
                "peak_source": peaks["source"] + " bf16_tflops (burst)",
                "flops_per_launch": g1_flops_launch, "avg_launch_ms": g1_launch_ms}
    # The SM clock the GEMM1 launches actually ran at (in-kernel clock64 / globaltimer, CTA 0,
    # averaged over launches; moe_stats.gemm1_sm_mhz) and the tensor-pipe efficiency at that
    # clock: achieved / (148 SMs x 8192 dense bf16 FLOP/clk/SM x clock).  8192 FLOP/clk/SM is
    # 2.25 PFLOP/s nominal at 1.856 GHz -- higher than 2.25 PF / 1.965 GHz (7737), so the
    # conservative per-cycle denominator.  Power management lowers the clock under dense MMA load.
    g1_mhz = st.get("gemm1_sm_mhz", 0.0)
    if g1_mhz > 0:
        per_clk_peak_tf = torch.cuda.get_device_properties(local).multi_processor_count * 8192.0 * g1_mhz * 1e6 / 1e12
        roofline["sm_mhz_in_kernel"] = g1_mhz
        roofline["peak_at_kernel_clock"] = per_clk_peak_tf
        roofline["frac_at_kernel_clock"] = achieved_tf / per_clk_peak_tf
        roofline["gemm2_sm_mhz_in_kernel"] = st.get("gemm2_sm_mhz", 0.0)
    h2d_gbs = st["h2d_weight_bytes"] / (st["h2d_ms"] * 1e-3) / 1e9 if st["h2d_ms"] > 0 else 0.0
    roofline_step = {"bound": "host_link" if t_io >= t_tc else "tensor",
                     "t_roofline_ms": t_roof * 1e3, "t_host_link_ms": t_io * 1e3,
                     "t_tensor_ms": t_tc * 1e3, "ms_per_step": ms, "frac": t_roof * 1e3 / ms,
                     "roofline_tokens_per_s": T / t_roof,
                     "host_link_probe_gbs_rank0": probe_gbs,
                     "host_link_probe_gbs_min": -allmax(-probe_gbs),
                     "host_link_probe_gbs_rank0_before_after": [probe_before, probe_after],
                     "h2d_achieved_gbs_in_copies_rank0": h2d_gbs,
                     "h2d_aggregate_gbs_over_step": step_weight_bytes / (ms * 1e-3) / 1e9,
                     "weight_bytes_per_step": step_weight_bytes,
                     "weight_bytes_per_rank": rank_bytes,
                     "algorithmic_weight_bytes_per_rank": alg_rank_bytes,
                     "expert_flops_per_step": work.expert_flops,
                     "oproj_flops_per_step": oproj_flops,
                     "tensor_peak_tflops": peaks["bf16_tflops_sustained"]}
    per_kernel_ms = {k: st[k] / args.steps for k in
                     ("h2d_ms", "route_ms", "permute_ms", "gemm1_ms", "gemm2_ms", "combine_ms",
                      "comm_ms", "oproj_ms", "norm_ms")}
    launches = allsum(st["kernel_launches"])

    # ---- e2e (pass 1's time; pass 2's copy-stream diagnostics)
    e2e = None
    if not args.no_e2e:
        tok_bytes = T * cfg.hidden * 2
        # The e2e step also moves its result device -> host while weights and the next tokens
        # stream in; on a shared host the two directions interfere.  Duplex probe: 1 GB H2D
        # with a concurrent D2H of the step's D2H : H2D ratio, best of 3 (CUDA events on the
        # H2D stream) -- the link bandwidth the e2e step can have.
        h2d_step = tok_bytes / world + step_weight_bytes / world
        ratio = (tok_bytes / world) / max(1.0, h2d_step)
        nb = 1 << 30
        hsrc = torch.empty(nb, dtype=torch.uint8).pin_memory()
        dbuf = torch.empty(nb, dtype=torch.uint8, device="cuda")
        nd = max(1 << 20, int(nb * ratio)) & ~15
        dsrc = torch.empty(nd, dtype=torch.uint8, device="cuda")
        hdst = torch.empty(nd, dtype=torch.uint8).pin_memory()
        s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
        duplex = 0.0
        for _ in range(3):
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(s_out):
                hdst.copy_(dsrc, non_blocking=True)
            with torch.cuda.stream(s_in):
                a.record(s_in)
                dbuf.copy_(hsrc, non_blocking=True)
                b.record(s_in)
            torch.cuda.synchronize()
            duplex = max(duplex, nb / (a.elapsed_time(b) * 1e-3) / 1e9)
        del hsrc, dbuf, dsrc, hdst
        duplex = -allmax(-duplex)
        # the step's link bandwidth is at most the plain H2D probe and at least what the duplex
        # probe saw; a duplex sample below what the step itself sustained is probe noise (the
        # step's D2H share is ~1% of its H2D at C1), so the ideal takes the better of the two
        link_gbs = max(duplex, -allmax(-probe_gbs))
        e2e_ideal_ms = h2d_step / (link_gbs * 1e9) * 1e3
        e2e = {"value": T / (ems / 1e3), "unit": "tokens/s", "ms_per_step": ems,
               "h2d_bytes_per_step": tok_bytes + step_weight_bytes,
               "h2d_token_bytes_per_step": tok_bytes, "h2d_weight_bytes_per_step": step_weight_bytes,
               "d2h_bytes_per_step": tok_bytes,
               "api": ("moe_taskb_forward2_host (two token partitions alpha/beta, one weight "
                       "stream)" if args.taskb and args.partitions == 2 else
                       "moe_taskb_forward_host (pinned host attention output / result, device "
                       "residual)" if args.taskb else
                       "moe_layer_forward_host (pinned host hidden/out)"),
               "copy_stream_ms_per_step_profile_pass": {
                   "weights": est["h2d_ms"] / args.steps, "tokens": est["h2d_token_ms"] / args.steps,
                   "note": "summed CUDA-event durations of the H2D copies (link busy time)"},
               "token_copy_latency_ms_profile_pass": {
                   "per_partition": [est["part_latency_ms"][p] / max(1, est["part_copies"][p])
                                     for p in range(2)],
                   "copies": est["part_copies"],
                   "note": "enqueue -> resident of each host token copy (partition 1 = beta)"},
               "matches_device_path": e2e_match,
               "link_roofline": {"h2d_gbs_duplex_probe": duplex, "d2h_to_h2d_ratio": ratio,
                                 "h2d_gbs_used": link_gbs,
                                 "ideal_ms_per_step": e2e_ideal_ms,
                                 "frac": e2e_ideal_ms / ems,
                                 "note": "H2D bytes per rank / the better of the plain H2D probe "
                                         "and the H2D bandwidth measured with the step's share of "
                                         "D2H running concurrently"}}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:   # the oracle baseline: N = 1 only
        os.sched_setaffinity(0, all_cpus)   # the oracle gets every host core
        cpu = cpu_baseline(layers[0], args.cpu_seconds, args.cpu_one_thread_tokens)

    # Per-expert rows of the last call on this rank (the load histogram goes with
    # every result; it is what makes DeepSeek-V2-Lite's grouped GEMMs uneven).
    routing = None
    try:
        layer.sync()
        dbg = layer.debug()

        class _Cai:
            def __init__(self, ptr, n):
                self.__cuda_array_interface__ = {"data": (int(ptr), False), "shape": (n,),
                                                 "typestr": "<i4", "version": 3}
        rows = torch.as_tensor(_Cai(dbg.counts, nl), device=f"cuda:{local}").cpu().tolist()
        mean = sum(rows) / max(1, len(rows))
        routing = {"rows_per_local_expert_last_call": rows,
                   "max_over_mean": max(rows) / mean if mean else None,
                   "min_over_mean": min(rows) / mean if mean else None}
    except Exception as e:  # noqa: BLE001 -- diagnostics only
        routing = {"error": str(e)}

    line = {"metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (seeded random bf16 weights/tokens shaped like the model)",
            "config": {"workload": cfg.name + (" GPU Task B (O-proj + RMSNorm + MoE)" if args.taskb else ""),
                       "tokens": T, "tokens_per_rank": Tr,
                       "hidden": cfg.hidden, "ffn": cfg.ffn, "experts": cfg.num_experts,
                       "experts_per_rank": nl, "top_k": cfg.top_k, "num_shared": cfg.num_shared,
                       "layers_cycled": args.layers, "staging_slots": st["num_slots"],
                       "experts_streamed_per_call": streamed,
                       "shared_experts": ("sharded" if shard else "replicated") if cfg.num_shared else None,
                       "packet_mb": args.packet_mb, "mover": bool(args.mover),
                       "l2": "inputs larger than L2: all expert weights re-streamed from host each step",
                       "parallelism": f"ep{world}", "ep_transport": transport,
                       "gpu_placement": placement,
                       "ep_comm_nranks": comm_nranks},
            "ms_per_step_profile_pass": ms_prof,
            "roofline": roofline, "roofline_step": roofline_step,
            "per_kernel_ms_per_step_rank0": per_kernel_ms,
            "e2e": e2e, "cpu_baseline": cpu, "clocks": clk,
            "gpu_launches": int(launches),
            "gpu_launches_per_step": launches / args.steps,
            "ms_per_step_dist_rank0": step_dist,
            "single_call_latency_ms": latency_ms,
            "host_affinity": affinity, "routing_rank0": routing}
    if rank == 0:
        print(json.dumps(line), flush=True)
    drop_layer(layer)
    for e in experts:
        e.close()
    if args.taskb:
        for hl in hls:
            hl.close()
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
