python -c "import paper_2504_09345_b200.build as b; b.build()" || exit 1
mkdir -p gpurun_out/p2p
for C in tiny mixtral_8x7b; do
MOE_BENCH_SHARE_GPU=1 timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 2 --warmup 1 --no-cpu --config $C > gpurun_out/p2p/bench_share2_$C.json 2> gpurun_out/p2p/bench_share2_$C.err
echo "rc=$? $C"; tail -c 700 gpurun_out/p2p/bench_share2_$C.json; echo; grep -i "error\|Traceback\|unavailable" gpurun_out/p2p/bench_share2_$C.err | head -5
done
