# full GPU suite (no -x) + smoke on HEAD
O=gpurun_out/r3o
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p $O
python __graft_entry__.py > $O/build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q --durations=5 > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
tail -3 $O/tests.log
timeout 300 python __graft_entry__.py smoke > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err; tail -c 300 $O/bench_default.json; echo
