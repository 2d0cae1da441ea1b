python -c "import paper_2504_09345_b200.build as b; b.build()" || exit 1
MOE_P2P_TRACE=1 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -s -k "ep_local and 8-shape3" 2>&1 | grep "\[p2p\]\|passed\|failed" | head -40
