# Every BASELINE.json workload on one B200 with the oracle leg ON (the oracle timed
# on the host cores beside the GPU for every config), plus the one-thread samples SURVEY names:
# all 64 tokens of C0 and a 256-token slice of C1.  usage: bash tools/gpu_allcfg.sh <outdir>
O=${1:-gpurun_out/allcfg}
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p $O
for C in tiny mixtral_8x7b mixtral_8x22b dbrx dsv2_lite; do
  OT=8
  [ $C = tiny ] && OT=64
  [ $C = mixtral_8x7b ] && OT=256
  timeout 1200 python bench.py --config $C --steps 20 --warmup 3 --cpu-one-thread-tokens $OT > $O/bench_$C.json 2> $O/bench_$C.err
  tail -1 $O/bench_$C.json | head -c 300; echo
done
