cd $GRAFT_REPO_ROOT
O=gpurun_out/r02q
mkdir -p $O
export TUNE_WARMUP=100
timeout 1200 python tools/tune.py --around "block=128 min_blocks=4,5,6" na6 cdp5ish hh_subset K_Pst NaTs2_t > $O/tune_occ.jsonl 2> $O/tune.err
