cd $GRAFT_REPO_ROOT
O=gpurun_out/r03g
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_nodes.py tests/test_gpu_column.py tests/test_gpu_fullsize.py -q -p no:cacheprovider -x > $O/gputests.log 2>&1; echo "pytest rc=$?" >> $O/gputests.log
for i in 1 2; do
timeout 300 python bench.py --workload column --cells 12500 --no-e2e --no-cpu --no-sustained > $O/col12k_$i.json 2> $O/col12k_$i.err
timeout 300 python bench.py --no-also --no-e2e --no-cpu --no-sustained > $O/syn10m_$i.json 2> $O/syn10m_$i.err
done
timeout 600 python bench.py --workload column --no-e2e --no-cpu --no-sustained > $O/col100k.json 2> $O/col100k.err
