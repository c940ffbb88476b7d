cd $GRAFT_REPO_ROOT
O=gpurun_out/r02w
mkdir -p $O
export TUNE_WARMUP=100
timeout 1200 python tools/tune.py --around "exp_smem=0,1 div_approx=0,1 recip=0,1" na6 > $O/tune_na6_relaxed.jsonl 2> $O/tune.err
timeout 900 python -m pytest tests/test_gpu_column.py -q -p no:cacheprovider -k errors > $O/gputests.log 2>&1; echo "rc=$?" >> $O/gputests.log
