# Round-2 GPU pass: GPU tests (all, with durations), then a short bench.  usage: bash tools/gpu_r2.sh <tag>
T=${1:-r2}
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${T}_smi.txt
timeout 2000 python -m pytest tests -m gpu -q ${PYTEST_ARGS:-} --durations=30 > gpurun_out/${T}_tests.log 2>&1; echo "tests_rc=$?" >> gpurun_out/${T}_tests.log
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
tail -3 gpurun_out/${T}_tests.log
