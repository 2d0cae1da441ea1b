"""CPU-side checks of the C-ABI library: it loads without a GPU, exports every symbol that
include/moe.h declares, validates configurations without touching CUDA, and packs experts in the
documented layout (host logic).  No compute calls are made here."""
import os
import re

import numpy as np
import pytest

import paper_2504_09345_b200 as moe
from paper_2504_09345_b200 import build as moe_build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    moe_build.build()
    return moe.load()


def test_library_exports_every_header_symbol(lib):
    header = open(os.path.join(ROOT, "include", "moe.h")).read()
    declared = set(re.findall(r"\b(moe_[a-z0-9_]+)\s*\(", header))
    assert declared, "no declarations parsed"
    assert declared == set(moe.EXPORTED)
    for name in declared:
        assert hasattr(lib, name), name


def test_library_has_no_hard_libcuda_dependency(lib):
    # static cudart; the driver is reached through cudaGetDriverEntryPoint at run time
    import subprocess
    out = subprocess.run(["ldd", moe.LIB_PATH], capture_output=True, text=True).stdout
    assert "libcuda.so" not in out and "libcudart.so" not in out


def test_packed_bytes_is_eq1_denominator(lib):
    # 6 * h * h_i bytes per expert (3 bf16 matrices)
    assert moe.moe_packed_expert_bytes(4096, 14336) == 352_321_536
    assert moe.moe_packed_expert_bytes(128, 256) == 196_608
    assert moe.moe_packed_expert_bytes(0, 256) == 0


def test_pack_expert_layout(lib):
    rng = np.random.default_rng(0)
    h, hi = 128, 384
    w1 = rng.integers(0, 65535, size=(hi, h), dtype=np.uint16)
    w3 = rng.integers(0, 65535, size=(hi, h), dtype=np.uint16)
    w2 = rng.integers(0, 65535, size=(h, hi), dtype=np.uint16)
    dst = np.zeros(6 * h * hi // 2, dtype=np.uint16)
    moe.moe_pack_expert(h, hi, w1, w3, w2, dst.ctypes.data)
    w13 = dst[: 2 * hi * h].reshape(2 * hi, h)
    for j in range(hi // 16):
        assert np.array_equal(w13[32 * j: 32 * j + 16], w1[16 * j: 16 * j + 16])
        assert np.array_equal(w13[32 * j + 16: 32 * j + 32], w3[16 * j: 16 * j + 16])
    assert np.array_equal(dst[2 * hi * h:].reshape(h, hi), w2)


def test_pack_rejects_bad_shapes(lib):
    a = np.zeros(10, dtype=np.uint16)
    with pytest.raises(moe.MoEError) as e:
        moe.moe_pack_expert(128, 200, a, a, a, a.ctypes.data)   # h_i % 128 != 0
    assert e.value.status == moe.MOE_E_UNSUPPORTED
    assert lib.moe_pack_expert(128, 256, None, None, None, None) == moe.MOE_E_INVAL


@pytest.mark.parametrize("kw,status", [
    (dict(top_k=9), moe.MOE_E_INVAL),                 # top_k > num_experts
    (dict(top_k=0), moe.MOE_E_INVAL),
    (dict(hidden=100), moe.MOE_E_UNSUPPORTED),        # h % 128 != 0
    (dict(ffn=200), moe.MOE_E_UNSUPPORTED),
    (dict(num_experts=200, top_k=2), moe.MOE_E_UNSUPPORTED),
    (dict(max_tokens=0), moe.MOE_E_INVAL),
    (dict(world_size=3), moe.MOE_E_UNSUPPORTED),      # 8 experts do not shard over 3 ranks
    (dict(rank=2, world_size=2), moe.MOE_E_INVAL),
    (dict(num_slots=1), moe.MOE_E_INVAL),             # double buffering needs >= 2 slots
    (dict(num_slots=33), moe.MOE_E_INVAL),            # > kMaxSlots
    (dict(num_slots=8), moe.MOE_E_INVAL),             # >= experts streamed per call (8)
    (dict(world_size=2, rank=0), moe.MOE_E_INVAL),    # EP needs an ncclUniqueId
])
def test_config_validation_without_gpu(lib, kw, status):
    base = dict(hidden=128, ffn=256, num_experts=8, top_k=2, num_shared=0, max_tokens=64,
                renormalize=1, device=0, world_size=1, rank=0, nccl_unique_id=None,
                packet_bytes=0, flags=0, num_slots=0)
    base.update(kw)
    cfg = moe.moe_config(**base)
    with pytest.raises(moe.MoEError) as e:
        moe.moe_init(cfg)
    assert e.value.status == status


def test_status_strings(lib):
    for s in range(8):
        assert moe.status_string(s).startswith("MOE_")


def test_header_compiles_as_plain_c99(tmp_path):
    """include/moe.h is a C ABI: it must compile as C99 with no C++ or CUDA types."""
    import shutil
    import subprocess
    if shutil.which("gcc") is None:
        import pytest
        pytest.skip("no gcc")
    src = tmp_path / "t.c"
    src.write_text('#include "moe.h"\nint main(void) { moe_stats s; moe_config c; (void)s; (void)c;'
                   ' return (int)MOE_FLAG_MOVER + (int)MOE_OK; }\n')
    inc = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include")
    r = subprocess.run(["gcc", "-std=c99", "-Wall", "-Wextra", "-Werror", "-pedantic",
                        "-fsyntax-only", "-I", inc, str(src)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


# ------------------------------------------------ MOE_FLAG_SHARD_SHARED host logic
@pytest.mark.parametrize("ffn,S,W", [(1408, 2, 8), (1408, 1, 8), (256, 2, 8), (384, 1, 8),
                                     (14336, 1, 2), (1408, 2, 2), (1408, 3, 4), (128, 1, 8)])
def test_shared_slice_partitions_the_concatenated_ffn(lib, ffn, S, W):
    """Slices of all ranks tile [0, S*ffn) in rank order with 128-column blocks, widths differ
    by at most one block (so every rank's slice fits one expert slot when S <= W)."""
    spans = [moe.moe_shared_slice(ffn, S, W, r) for r in range(W)]
    pos = 0
    for c0, w in spans:
        assert c0 == pos and w % 128 == 0 and w >= 0
        pos += w
    assert pos == S * ffn
    widths = [w for _, w in spans]
    assert max(widths) - min(widths) <= 128
    if S <= W:
        assert max(widths) <= ffn


def test_shared_slice_rejects_bad_arguments(lib):
    for args in ((1408, 0, 8, 0), (1408, 2, 0, 0), (1408, 2, 8, 8), (1408, 2, 8, -1),
                 (100, 2, 8, 0)):
        with pytest.raises(moe.MoEError) as ei:
            moe.moe_shared_slice(*args)
        assert ei.value.status == moe.MOE_E_INVAL


def test_shared_slices_sum_to_the_shared_ffns():
    """The math the sharded layout relies on (include/moe.h MOE_FLAG_SHARD_SHARED): the sum over
    ranks of the SwiGLU FFN of each rank's slice (shared_slice_weights) equals the sum of the
    S shared experts' FFNs, in fp64 on bf16 weights -- pins the slicing (rows of W1/W3, columns
    of W2, expert boundaries crossed by a slice) against whole experts."""
    import synth
    from paper_2504_09345_b200 import shared_slice_weights
    cfg = synth.MoEConfig("custom", 19, 256, 384, 4, 2, 8, 3)
    inp = synth.gen_inputs(cfg)
    f64 = lambda a: synth.bf16_bits_to_f32(a).astype(np.float64)
    x = f64(inp.x)

    def ffn(w1, w3, w2):
        a, b = x @ f64(w1).T, x @ f64(w3).T
        return (a / (1 + np.exp(-a)) * b) @ f64(w2).T

    ne = cfg.num_experts
    want = sum(ffn(inp.w1[ne + s], inp.w3[ne + s], inp.w2[ne + s]) for s in range(cfg.num_shared))
    for W in (3, 4, 8):
        parts = [shared_slice_weights(cfg.ffn, inp.w1[ne:], inp.w3[ne:], inp.w2[ne:], W, r)
                 for r in range(W)]
        got = sum(ffn(*p) for p in parts if p is not None)
        np.testing.assert_allclose(got, want, rtol=1e-12, atol=1e-12)


def test_shard_shared_rejected_outside_its_envelope(lib):
    """MOE_FLAG_SHARD_SHARED needs the P2P transport, W > 1 and 1 <= num_shared <= W; moe_init
    refuses anything else before touching CUDA."""
    for kw in (dict(world_size=1, local_ep=True, num_shared=1),
               dict(world_size=2, local_ep=True, num_shared=3),
               dict(world_size=2, local_ep=True, num_shared=0),
               dict(world_size=2, num_shared=1)):               # NCCL transport
        with pytest.raises(moe.MoEError) as ei:
            moe.MoELayer(256, 256, 8, 2, 64, nccl_unique_id=b"k" * 128, shard_shared=True, **kw)
        assert ei.value.status == moe.MOE_E_UNSUPPORTED, kw


def build_c_example(tmpdir) -> str:
    """examples/moe_layer.c: the C ABI from plain C99 (no Python) -- compiled and linked here;
    tests/test_gpu_parity.py runs it on the GPU against the oracle."""
    import subprocess
    exe = os.path.join(str(tmpdir), "moe_layer")
    pkg = os.path.join(ROOT, "paper_2504_09345_b200")
    cmd = ["gcc", "-std=c99", "-O2", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"),
           "-I", "/usr/local/cuda/include", os.path.join(ROOT, "examples", "moe_layer.c"),
           "-L", pkg, "-lmoe_b200", "-Wl,-rpath," + pkg, "-L", "/usr/local/cuda/lib64", "-lcudart",
           "-Wl,-rpath,/usr/local/cuda/lib64", "-o", exe]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_c_example_builds(lib, tmp_path):
    exe = build_c_example(tmp_path)
    assert os.path.exists(exe)
