cd $GRAFT_REPO_ROOT
O=gpurun_out/r02j
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_nodes.py tests/test_gpu_column.py -q -p no:cacheprovider -x > $O/gputests.log 2>&1; echo "pytest rc=$?" >> $O/gputests.log
export TUNE_WARMUP=30 TUNE_N=1250000 TUNE_NODES=262500
timeout 900 python tools/tune.py --around "ilp=1,2 tile=1024,2304 min_blocks=3,4" ProbAMPANMDA_EMS > $O/tune_syn_small.jsonl 2> $O/tune.err
for cells in 100000 12500; do
timeout 600 python bench.py --workload column --cells $cells --no-e2e --no-cpu --no-sustained > $O/col_${cells}.json 2> $O/col_${cells}.err
done
