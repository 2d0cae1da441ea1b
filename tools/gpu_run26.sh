mkdir -p gpurun_out/r26
python -c "import paper_2504_09345_b200.build as b; b.build()" || exit 1
timeout 1200 python -m pytest tests/test_gpu_fuzz.py -q 2>&1 | tail -5 | tee gpurun_out/r26/pytest_fuzz.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2 | tee gpurun_out/r26/smoke.log
