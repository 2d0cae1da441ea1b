set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
nproc; lscpu | grep -E "Model name|Socket|NUMA node\(s\)|^CPU\(s\)"
nvidia-smi topo -m | head -5
timeout 900 python -m pytest tests -m gpu -x -q -k "not full_size" 2>&1 | tail -40
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -5
