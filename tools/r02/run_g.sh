cd $GRAFT_REPO_ROOT
O=gpurun_out/r02g
mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rs --durations=10 > $O/gputests.log 2>&1; echo "pytest rc=$?" >> $O/gputests.log
timeout 300 python __graft_entry__.py smoke > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
for cells in 100000 12500; do
NMODL_COLUMN_MODE=grouped timeout 600 python bench.py --workload column --cells $cells --no-e2e --no-cpu --no-sustained > $O/col_${cells}.json 2> $O/col_${cells}.err
done
for c in 1 2 4 8; do
NMODL_E2E_CHUNKS=$c timeout 600 python bench.py --no-also --no-cpu --no-sustained > $O/syn_chunks$c.json 2> $O/syn_chunks$c.err
done
