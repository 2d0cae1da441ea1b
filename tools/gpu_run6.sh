set -x
timeout 900 python -m pytest tests -m gpu -x -q -k "ragged or tiny or ep_path" 2>&1 | tail -3
timeout 900 python -m paper_2504_09345_b200.profiler --config mixtral_8x7b --tokens 4096,16384,65536,131072 > gpurun_out/profiler_c1_b.json 2>gpurun_out/profiler_c1_b.err; cat gpurun_out/profiler_c1_b.json; tail -3 gpurun_out/profiler_c1_b.err
