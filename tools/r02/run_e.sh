cd $GRAFT_REPO_ROOT
O=gpurun_out/r02e
mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=15 > $O/gputests.log 2>&1; echo "pytest rc=$?" >> $O/gputests.log
timeout 300 python __graft_entry__.py smoke > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
export PROFILE_TAG=r02e_prof
timeout 1500 python tools/profile_bench.py $O/prof > $O/profile.log 2>&1; echo "rc=$?" >> $O/profile.log
cp $O/prof/ncu_traffic.json profiles/ncu_traffic.json
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
timeout 600 python bench.py --workload column > $O/bench_column.json 2> $O/bench_column.err; echo "rc=$?" >> $O/bench_column.err
