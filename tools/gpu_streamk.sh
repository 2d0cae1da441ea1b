# Stream-K last wave (MOE_GEMM_STREAMK) check: GEMM parity tests, then C1 / DBRX / C4 benches
# with it off / on (GEMM1 / GEMM2 ms per step, in-kernel clock).  usage: bash tools/gpu_streamk.sh <tag>
T=${1:-sk}
O=gpurun_out/$T; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q -k "streamk or tile_variants or taskb_gemm_variants or full_size" 2>&1 | tail -3
for C in ${SKCFG:-mixtral_8x7b dbrx dsv2_lite mixtral_8x22b}; do
  for SK in 0 1; do
    MOE_GEMM_STREAMK=$SK timeout 600 python bench.py --config $C --steps 10 --warmup 3 --no-cpu --no-e2e > $O/bench_${C}_sk$SK.json 2> $O/bench_${C}_sk$SK.err
    python - <<PY
import json
d = json.load(open("$O/bench_${C}_sk$SK.json"))
k = d["per_kernel_ms_per_step_rank0"]; r = d["roofline"]
print("$C streamk=$SK", round(d["value"]), "step", round(d["roofline_step"]["frac"], 4),
      "g1", round(k["gemm1_ms"], 3), "g2", round(k["gemm2_ms"], 3), "frac", round(r["frac"], 4),
      "mhz", round(r.get("sm_mhz_in_kernel", 0)), "frac@clk", round(r.get("frac_at_kernel_clock", 0), 4))
PY
  done
done
