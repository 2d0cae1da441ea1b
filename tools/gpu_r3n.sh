# permute with 8 vectors in flight and register-resident destinations: full GPU suite + C1 / C4 bench lines
O=gpurun_out/r3n
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p $O
python __graft_entry__.py > $O/build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x --durations=5 > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
tail -3 $O/tests.log
timeout 900 python bench.py --no-cpu > $O/bench_c1.json 2> $O/bench_c1.err; tail -c 200 $O/bench_c1.json; echo
timeout 900 python bench.py --config dsv2_lite --no-cpu > $O/bench_dsv2.json 2> $O/bench_dsv2.err; tail -c 200 $O/bench_dsv2.json; echo
timeout 900 python bench.py --tokens 131072 --steps 10 --warmup 3 --no-cpu --no-e2e > $O/bench_131k.json 2> $O/bench_131k.err; tail -c 200 $O/bench_131k.json; echo
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"permute|combine" --csv --log-file $O/permute_combine_c1.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"permute|combine" -c 4 --csv --log-file $O/permute_combine_c4.csv python bench.py --config dsv2_lite --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
ls $O
