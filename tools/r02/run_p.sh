cd $GRAFT_REPO_ROOT
O=gpurun_out/r02p
mkdir -p $O
export TUNE_WARMUP=30
timeout 900 python tools/tune.py --around "pipe=0,1 min_blocks=3,4 tile=1152,2304" ProbAMPANMDA_EMS > $O/tune_syn_pipe.jsonl 2> $O/tune.err
timeout 600 python tools/tune.py --around "ilp=1,2 min_blocks=0,2" hh_subset > $O/tune_hh_ilp.jsonl 2>> $O/tune.err
timeout 900 python tools/tune.py --around "exp_smem=0,1 exp_share=0,1 quot=0,1 ilp=1,2" K_Pst > $O/tune_kpst2.jsonl 2>> $O/tune.err
timeout 600 python tools/tune.py --around "ilp=1,2 min_blocks=0,2 pipe=0,1" Ih cadyn SKv3_1 > $O/tune_small.jsonl 2>> $O/tune.err
