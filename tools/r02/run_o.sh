cd $GRAFT_REPO_ROOT
O=gpurun_out/r02o
mkdir -p $O
export TUNE_WARMUP=30
timeout 1200 python tools/tune.py --around "fast_path=0,1 div_approx=0,1 exp_share=0,1 recip=0,1" ProbAMPANMDA_EMS > $O/tune_syn_relaxed.jsonl 2> $O/tune.err
timeout 600 python tools/tune.py --around "fast_path=1 fast_redo=1 min_blocks=3,4" ProbAMPANMDA_EMS >> $O/tune_syn_relaxed.jsonl 2>> $O/tune.err
