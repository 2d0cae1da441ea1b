# router edge shapes + routing tests on HEAD
O=gpurun_out/r3m
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p $O
python __graft_entry__.py > $O/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "router or special or tie" > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
tail -5 $O/tests.log
