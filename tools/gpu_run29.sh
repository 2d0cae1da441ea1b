python -c "import paper_2504_09345_b200.build as b; b.build()" || exit 1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "ep_local and 8-shape3" 2>&1 | grep -v "^\s*$" | grep -i "error\|assert\|moe\|rank" | head -30
