set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "ep_local or ep_path" 2>&1 | tail -15
timeout 900 python -m pytest tests -m gpu -x -q -k "not full_size" 2>&1 | tail -3
timeout 600 compute-sanitizer --tool memcheck --error-exitcode 9 python __graft_entry__.py smoke > gpurun_out/sanitizer_memcheck.log 2>&1; echo "memcheck rc=$?"; tail -3 gpurun_out/sanitizer_memcheck.log
timeout 600 compute-sanitizer --tool racecheck --error-exitcode 9 python __graft_entry__.py smoke > gpurun_out/sanitizer_racecheck.log 2>&1; echo "racecheck rc=$?"; tail -3 gpurun_out/sanitizer_racecheck.log
timeout 600 compute-sanitizer --tool synccheck --error-exitcode 9 python __graft_entry__.py smoke > gpurun_out/sanitizer_synccheck.log 2>&1; echo "synccheck rc=$?"; tail -3 gpurun_out/sanitizer_synccheck.log
