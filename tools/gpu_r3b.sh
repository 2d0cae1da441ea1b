# router v7 sweep + the router-variant parity tests
bash tools/gpu_router_v7.sh gpurun_out/router7c
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "router_experts_per_warp" > gpurun_out/router7c/tests.log 2>&1; tail -3 gpurun_out/router7c/tests.log
