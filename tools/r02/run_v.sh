cd $GRAFT_REPO_ROOT
O=gpurun_out/r02v
mkdir -p $O
export TUNE_WARMUP=100
timeout 1200 python tools/tune.py --around "fast_path=0,1 lu_spec=0,1 pipe=0,1" na6 cdp5ish > $O/tune_kin_fp.jsonl 2> $O/tune.err
