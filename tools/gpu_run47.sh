python -c "import paper_2504_09345_b200.build as b; b.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_fuzz.py -q -k "maxima" 2>&1 | tail -5
