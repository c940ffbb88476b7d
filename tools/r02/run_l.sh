cd $GRAFT_REPO_ROOT
O=gpurun_out/r02l
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "reciprocal or speculative" > $O/gputests.log 2>&1; echo "pytest rc=$?" >> $O/gputests.log
export TUNE_WARMUP=100
timeout 900 python tools/tune.py --around "lu_rcp=0,1 min_blocks=0,2" na6 cdp5ish > $O/tune_kin.jsonl 2> $O/tune.err
for cells in 100000 12500; do
timeout 600 python bench.py --workload column --cells $cells --no-e2e --no-cpu > $O/col_${cells}.json 2> $O/col_${cells}.err
done
