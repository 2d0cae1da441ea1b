# Contiguous Data Mover (MOE_FLAG_MOVER) check: its GPU tests, then C1 / C4 benches with the
# mover (one and two packets in flight) beside the event-ordered engine.  usage: bash tools/gpu_mover.sh <tag>
T=${1:-mover}
O=gpurun_out/$T; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_mover.py -x -q -s 2>&1 | grep -v "^$" | tail -8
for C in mixtral_8x7b dsv2_lite; do
  for V in "off 1" "on 1" "on 2"; do
    set -- $V
    F=""; [ $1 = on ] && F="--mover"
    MOE_MOVER_INFLIGHT=$2 timeout 600 python bench.py --config $C --steps 10 --warmup 3 --no-cpu $F > $O/bench_${C}_$1$2.json 2> $O/bench_${C}_$1$2.err
    python - <<PY
import json
d = json.load(open("$O/bench_${C}_$1$2.json"))
e = d.get("e2e") or {}
print("$C mover=$1 inflight=$2", round(d["value"]), "step", round(d["roofline_step"]["frac"], 4),
      "e2e", round(e.get("value", 0)), "h2d_gbs", round(d["roofline_step"]["h2d_achieved_gbs_in_copies_rank0"], 2))
PY
  done
done
