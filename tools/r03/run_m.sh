cd $GRAFT_REPO_ROOT
O=gpurun_out/r03m
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -rs > $O/gputests.log 2>&1; echo "pytest rc=$?" >> $O/gputests.log
for i in 1 2; do
timeout 600 python bench.py --no-cpu --no-e2e --no-sustained > $O/bench_$i.json 2> $O/bench_$i.err
done
