"""NEXT-1 pipeline profiler on the GPU (§6.3): sweep the token
count through the real layer, fit GPU time vs tokens, measure the per-layer weight transfer, and
solve for n_real -- the token count at which the GPU time line meets the transfer time."""
import pytest

import synth
from paper_2504_09345_b200 import ledger, profiler

pytestmark = pytest.mark.gpu


def test_profiler_small_layer_n_real_near_eq2():
    """h = 1024, h_i = 2048, 8 experts, top-2 (100.7 MB of expert weights per layer), swept over
    16k..128k tokens.  The paper's procedure must give (1) a line that fits every point within
    5% (GPU time is linear in n above a few waves), (2) a per-layer transfer time within 15% of
    the layer's bytes over the paper's 1 GB probe bandwidth, and (3) n_real within
    0.5x..1.5x of Eq. 2's n = (C / B) (N_e / N_k) with the measured peaks."""
    cfg = synth.MoEConfig("profiler_small", 30, 1024, 2048, 8, 2, 131072)
    res = profiler.profile(cfg, [16384, 32768, 65536, 131072], steps=3)
    print(res)
    for p in res["points"]:
        assert abs(p["fit_rel_residual"]) <= 0.05, p
    bytes_ = ledger.expert_bytes(cfg.hidden, cfg.ffn) * cfg.num_experts
    t_link = bytes_ / (res["eq2_inputs"]["host_link_gbs"] * 1e9) * 1e3
    # the sweep's copies overlap the GEMMs of up to 131k tokens (power-capped clocks, HBM traffic);
    # one box measured them 10% slower than the idle 1-GB probe, others within 5%
    assert abs(res["t_io_ms"] - t_link) <= 0.15 * t_link, (res["t_io_ms"], t_link)
    assert 0.5 * res["n_eq2_estimate"] <= res["n_real"] <= 1.5 * res["n_eq2_estimate"], res
