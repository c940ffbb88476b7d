cd $GRAFT_REPO_ROOT
O=gpurun_out/r02r
mkdir -p $O
export TUNE_WARMUP=100
timeout 1200 python tools/tune.py --around "ilp=2 min_blocks=0,1,2 pipe=0,1" na6 cdp5ish > $O/tune_kin_ilp2.jsonl 2> $O/tune.err
