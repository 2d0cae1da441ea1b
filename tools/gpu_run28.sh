mkdir -p gpurun_out/p2p
python -c "import paper_2504_09345_b200.build as b; b.build()" || exit 1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "ep_local or ep_path or tiny or host" 2>&1 | tail -5 | tee gpurun_out/p2p/pytest_local.log
timeout 900 python -m pytest tests/test_gpu_ep_ipc.py -x -q 2>&1 | tail -25 | tee gpurun_out/p2p/pytest_ipc.log
