cd $GRAFT_REPO_ROOT
O=gpurun_out/r03e
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_nodes.py -k combine -q -p no:cacheprovider > $O/gputests.log 2>&1; echo "pytest rc=$?" >> $O/gputests.log
for i in 1 2; do
for p in -1 0; do
NMODL_GROUP_PRIO=$p timeout 300 python bench.py --workload column --cells 12500 --no-e2e --no-cpu --no-sustained > $O/col12k_prio${p}_$i.json 2> $O/col12k_prio${p}_$i.err
done
done
NMODL_GROUP_PRIO=-1 timeout 600 python bench.py --workload column --no-e2e --no-cpu --no-sustained > $O/col100k_prio-1.json 2> $O/col100k_prio-1.err
