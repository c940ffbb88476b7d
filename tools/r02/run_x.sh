cd $GRAFT_REPO_ROOT
O=gpurun_out/r02x
mkdir -p $O
export TUNE_WARMUP=100
timeout 1200 python tools/tune.py --around "fmad=0,1" na6 cdp5ish hh_subset K_Pst NaTs2_t Ca_HVA > $O/tune_fmad.jsonl 2> $O/tune.err
