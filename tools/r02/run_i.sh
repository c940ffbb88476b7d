cd $GRAFT_REPO_ROOT
O=gpurun_out/r02i
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_nodes.py tests/test_gpu_column.py -q -p no:cacheprovider -x > $O/gputests.log 2>&1; echo "pytest rc=$?" >> $O/gputests.log
for c in 1 2 4; do
NMODL_E2E_CHUNKS=$c timeout 600 python bench.py --no-also --no-cpu --no-sustained --steps 20 > $O/syn_chunks$c.json 2> $O/syn_chunks$c.err
done
for cells in 100000 12500; do
for mode in overlap grouped; do
NMODL_COLUMN_MODE=$mode timeout 600 python bench.py --workload column --cells $cells --no-e2e --no-cpu --no-sustained > $O/col_${cells}_${mode}.json 2> $O/col_${cells}_${mode}.err
done
done
