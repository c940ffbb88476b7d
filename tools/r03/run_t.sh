cd $GRAFT_REPO_ROOT
O=gpurun_out/r03t
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_column.py -q -p no:cacheprovider -x > $O/gputests.log 2>&1; echo "pytest rc=$?" >> $O/gputests.log
for i in 1 2; do
for m in chained grouped; do
NMODL_COLUMN_MODE=$m timeout 300 python bench.py --workload column --cells 12500 --no-e2e --no-cpu --no-sustained > $O/col12k_${m}_$i.json 2> $O/col12k_${m}_$i.err
done
done
for m in chained grouped; do
NMODL_COLUMN_MODE=$m timeout 600 python bench.py --workload column --no-e2e --no-cpu --no-sustained > $O/col100k_$m.json 2> $O/col100k_$m.err
done
