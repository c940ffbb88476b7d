cd $GRAFT_REPO_ROOT
O=gpurun_out/r02y
mkdir -p $O
export TUNE_WARMUP=100 TUNE_N=10000000
timeout 1200 python tools/tune.py --around "min_blocks=2" na6 cdp5ish > $O/tune_kin_10m.jsonl 2> $O/tune.err
