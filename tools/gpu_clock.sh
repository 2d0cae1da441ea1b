# SM clock inside the expert GEMMs (moe_stats.gemm1_sm_mhz) for the default engine and the GEMM
# variants, C1 and DBRX; plus the GPU test suite.  usage: bash tools/gpu_clock.sh <tag>
T=${1:-clk}
O=gpurun_out/$T; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for C in mixtral_8x7b dbrx; do
  for V in "-1 0 0" "1 0 0" "1 1 0" "1 0 1" "0 0 0"; do
    set -- $V
    MOE_GEMM_PAIR=$1 MOE_GEMM_ALT=$2 MOE_GEMM_TAILSWAP=$3 timeout 600 python bench.py --config $C --steps 10 --warmup 3 --no-cpu --no-e2e > $O/bench_${C}_$1$2$3.json 2> $O/bench_${C}_$1$2$3.err
    python - <<PY
import json
d = json.load(open("$O/bench_${C}_$1$2$3.json"))
k = d["per_kernel_ms_per_step_rank0"]; r = d["roofline"]
print("$C pair=$1 alt=$2 tailswap=$3", round(d["value"]), "step", round(d["roofline_step"]["frac"], 4),
      "g1", round(k["gemm1_ms"], 3), "g2", round(k["gemm2_ms"], 3), "frac", round(r["frac"], 4),
      "mhz", round(r.get("sm_mhz_in_kernel", 0)), "g2mhz", round(r.get("gemm2_sm_mhz_in_kernel", 0)), "frac@clk", round(r.get("frac_at_kernel_clock", 0), 4))
PY
  done
done
