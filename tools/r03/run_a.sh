cd $GRAFT_REPO_ROOT
O=gpurun_out/r03a
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -rs -x > $O/gputests.log 2>&1; echo "pytest rc=$?" >> $O/gputests.log
timeout 300 python __graft_entry__.py smoke > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
for w in 1 2 3 4 6; do
  NMODL_NODE_WAVES=$w timeout 300 python bench.py --workload column --cells 12500 --no-e2e --no-cpu --no-sustained > $O/col12k_w$w.json 2> $O/col12k_w$w.err
done
for mb in 3 5 6; do
  NMODL_OPT_ProbAMPANMDA_EMS="min_blocks=$mb" timeout 300 python bench.py --workload column --cells 12500 --no-e2e --no-cpu --no-sustained > $O/col12k_mb$mb.json 2> $O/col12k_mb$mb.err
done
NMODL_COLUMN_CELLS=12500 timeout 900 python tools/profile_bench.py $O/prof12k column > $O/prof12k.log 2>&1; echo "rc=$?" >> $O/prof12k.log
timeout 600 python bench.py --workload column > $O/bench_column.json 2> $O/bench_column.err; echo "rc=$?" >> $O/bench_column.err
