python -c "import paper_2504_09345_b200.build as b; b.build()" || exit 1
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -4
