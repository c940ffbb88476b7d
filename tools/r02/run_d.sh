cd $GRAFT_REPO_ROOT
O=gpurun_out/r02d
mkdir -p $O
export TUNE_WARMUP=50
timeout 600 python tools/tune.py --around "min_blocks=0,3,4 tile=2048,2304" ProbAMPANMDA_EMS > $O/tune_syn.jsonl 2> $O/tune.err
timeout 600 python tools/tune.py --around "min_blocks=0,3 block=128,256" hh_subset > $O/tune_hh.jsonl 2>> $O/tune.err
timeout 600 python tools/tune.py --around "min_blocks=0,2,3" na6 cdp5ish > $O/tune_kin.jsonl 2>> $O/tune.err
timeout 600 python tools/tune.py --around "ilp=1,2 min_blocks=0,2,3" K_Pst > $O/tune_kpst.jsonl 2>> $O/tune.err
