"""Ledger / roofline arithmetic pinned to numbers the paper prints (tests/golden/paper_numbers.json)."""
import json
import os

import pytest

from paper_2504_09345_b200 import ledger as L

G = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_numbers.json")))


@pytest.mark.parametrize("gpu", ["A40", "L40", "A100"])
def test_table2_reproduces_with_binary_prefixes(gpu):
    t = G["table2"]
    n = L.eq2_tokens_to_saturate(t["gpus"][gpu], t["B"], t["N_e"], t["N_k"])
    # printed to 0.1k; A100's 39,936 is printed as 40.0k (within one printed digit)
    assert abs(n / 1000 - t["tokens_k"][gpu]) <= 0.1
    kv = L.kv_bytes_per_token(32, 4096, 4)
    assert kv == 131072
    for seq, key in ((256, "kv_gb_seq256"), (512, "kv_gb_seq512")):
        gb = n * seq * kv / 2 ** 20 / 1000       # MiB / 1000, truncated (reading R15)
        printed = t[key][gpu]
        if gpu == "A100" and seq == 512:
            assert abs(gb - printed) / printed < 1e-3   # 2555.9 vs printed 2554
        else:
            assert int(gb) == printed


def test_eq2_text_example():
    # "requires processing 19,200 tokens in parallel"
    assert L.eq2_tokens_to_saturate(150, 32, 8, 2) == 19200


@pytest.mark.parametrize("name", ["mixtral_8x7b", "mixtral_8x22b", "dbrx"])
def test_model_sizes_from_eq1_denominator(name):
    m = G["model_sizes_gb"][name]
    b = L.model_bytes(m["layers"], m["N_e"], m["h"], m["hi"], m["s"], m["vocab"])
    assert abs(b / 1e9 - m["gb"]) / m["gb"] < 0.01
    assert abs(b / 2 / 1e9 - m["params_b"]) / m["params_b"] < 0.01


def test_eq1_forms_and_limits():
    ex = G["eq1_example"]
    r = L.eq1_intensity(ex["n"], 8, 2, 4096, 14336, 4, form="right")
    assert abs(r - ex["value"]) / ex["value"] < ex["rel_tol"]
    for form in ("left", "right"):
        assert L.eq1_intensity(1, 8, 8, 4096, 14336, 4, form) == pytest.approx(1.0)
        assert L.eq1_intensity(2000, 8, 2, 4096, 14336, 4, form) == pytest.approx(
            2 * L.eq1_intensity(1000, 8, 2, 4096, 14336, 4, form))
        # large-m limit -> n N_k / N_e
        assert L.eq1_intensity(1000, 8, 2, 128, 128 * 10 ** 6, 4, form) == pytest.approx(250, rel=1e-5)


def test_delta_weight_transfer_time():
    d = G["delta_seconds"]
    delta = d["model_gb"] / d["b_io_gbs"]
    assert delta == pytest.approx(4.82, abs=0.01) and abs(delta - d["approx_s"]) < 0.25


def test_layer_work_mixtral():
    w = L.layer_work(4096, 4096, 14336, 8, 2)
    assert w.weight_bytes == 8 * 352_321_536
    assert w.expert_flops == 4096 * 2 * 6 * 4096 * 14336
    assert w.gemm1_flops + w.gemm2_flops == w.expert_flops
    r = L.roofline_time_s(w, 2250, 55)
    assert r["bound"] == "host_link" and r["t_host_link_s"] == pytest.approx(0.05125, rel=1e-3)
