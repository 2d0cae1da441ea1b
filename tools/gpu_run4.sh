set -x
timeout 1200 python -m pytest tests -m gpu -x -q -k "not full_size" 2>&1 | tail -30
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu 2>&1 | tail -3
