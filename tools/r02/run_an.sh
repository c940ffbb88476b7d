cd $GRAFT_REPO_ROOT
O=gpurun_out/r02an
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_column.py tests/test_gpu_nodes.py -q -p no:cacheprovider -x > $O/gputests.log 2>&1; echo "rc=$?" >> $O/gputests.log
for cells in 100000 12500; do
timeout 600 python bench.py --workload column --cells $cells --no-e2e --no-cpu > $O/col_${cells}.json 2> $O/col_${cells}.err
done
timeout 600 python bench.py --no-also --no-e2e --no-cpu > $O/syn.json 2> $O/syn.err
