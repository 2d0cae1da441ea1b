# combine with 4 row vectors in flight for top-1/2: full GPU suite + combine ncu at C1 / C4 + C1 bench
O=gpurun_out/r3p
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p $O
python __graft_entry__.py > $O/build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q --durations=5 > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
tail -3 $O/tests.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"permute|combine" --csv --log-file $O/permute_combine_c1.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"permute|combine" -c 4 --csv --log-file $O/permute_combine_c4.csv python bench.py --config dsv2_lite --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err; tail -c 300 $O/bench_default.json; echo
