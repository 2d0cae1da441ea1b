python -c "import paper_2504_09345_b200.build as b; b.build()" || exit 1
mkdir -p gpurun_out/profiler2
timeout 1200 python -m paper_2504_09345_b200.profiler --config mixtral_8x7b --tokens 4096,16384,32768,65536,98304,131072 --steps 3 > gpurun_out/profiler2/profiler_mixtral_8x7b.json 2> gpurun_out/profiler2/p1.err
timeout 1200 python -m paper_2504_09345_b200.profiler --config dsv2_lite --tokens 32768,65536,131072,196608 --steps 3 > gpurun_out/profiler2/profiler_dsv2_lite.json 2> gpurun_out/profiler2/p2.err
python -m paper_2504_09345_b200.perfmodel validate gpurun_out/profiler2/profiler_mixtral_8x7b.json > gpurun_out/profiler2/perfmodel_validation_mixtral.json
python -m paper_2504_09345_b200.perfmodel validate gpurun_out/profiler2/profiler_dsv2_lite.json > gpurun_out/profiler2/perfmodel_validation_dsv2.json
tail -c 600 gpurun_out/profiler2/profiler_mixtral_8x7b.json; echo; tail -c 600 gpurun_out/profiler2/profiler_dsv2_lite.json; echo
grep -i "accuracy" gpurun_out/profiler2/perfmodel_validation_*.json
