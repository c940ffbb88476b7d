cd $GRAFT_REPO_ROOT
O=gpurun_out/r02c
mkdir -p $O
./tools/micro/flush_modes > $O/flush_modes.jsonl 2>&1
./tools/micro/fp64_peak > $O/fp64_peak.jsonl 2>&1
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
timeout 600 python bench.py --workload column > $O/bench_column.json 2> $O/bench_column.err; echo "rc=$?" >> $O/bench_column.err
timeout 1500 python tools/profile_bench.py $O/prof > $O/profile.log 2>&1; echo "rc=$?" >> $O/profile.log
