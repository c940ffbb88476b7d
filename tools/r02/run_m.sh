cd $GRAFT_REPO_ROOT
O=gpurun_out/r02m
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_column.py tests/test_gpu_parity.py -q -p no:cacheprovider -k "column or speculative or lu" > $O/gputests.log 2>&1; echo "pytest rc=$?" >> $O/gputests.log
for cells in 100000 12500; do
for mode in grouped grouped_ih; do
NMODL_COLUMN_MODE=$mode timeout 600 python bench.py --workload column --cells $cells --no-e2e --no-cpu > $O/col_${cells}_${mode}.json 2> $O/col_${cells}_${mode}.err
done
done
export PROFILE_TAG=r02k_prof
cp profiles/ncu_traffic.json $O/ncu_traffic.json
mkdir -p $O/prof && cp profiles/ncu_traffic.json $O/prof/ncu_traffic.json
timeout 900 python tools/profile_bench.py $O/prof kinetic1m > $O/profile.log 2>&1; echo "rc=$?" >> $O/profile.log
