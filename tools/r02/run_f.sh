cd $GRAFT_REPO_ROOT
O=gpurun_out/r02f
mkdir -p $O
./tools/micro/store_hints > $O/store_hints.jsonl 2>&1
timeout 900 python -m pytest tests/test_gpu_column.py tests/test_gpu_nccl.py -q -p no:cacheprovider -rs > $O/gputests.log 2>&1; echo "pytest rc=$?" >> $O/gputests.log
for cells in 100000 12500; do
for mode in grouped concurrent sequential; do
NMODL_COLUMN_MODE=$mode timeout 600 python bench.py --workload column --cells $cells --no-e2e --no-cpu --no-sustained --steps 200 --warmup 20 > $O/col_${cells}_${mode}.json 2> $O/col_${cells}_${mode}.err
done
done
