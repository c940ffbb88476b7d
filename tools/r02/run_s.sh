cd $GRAFT_REPO_ROOT
O=gpurun_out/r02s
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_nodes.py tests/test_gpu_column.py tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "unique or column or node or one_instance" > $O/gputests.log 2>&1; echo "pytest rc=$?" >> $O/gputests.log
for cells in 100000 12500; do
timeout 600 python bench.py --workload column --cells $cells --no-e2e --no-cpu > $O/col_${cells}.json 2> $O/col_${cells}.err
done
./tools/micro/lu_lanes > $O/lu_lanes.json 2>&1
