cd $GRAFT_REPO_ROOT
O=gpurun_out/r03w
mkdir -p $O
timeout 600 python tools/tune.py --around "grid_waves=0,1,2,4" hh_subset >> $O/tune.jsonl 2>> $O/tune.err
TUNE_N=3333333 timeout 900 python tools/tune.py --around "grid_waves=0,1,2,4" K_Pst NaTs2_t >> $O/tune.jsonl 2>> $O/tune.err
timeout 600 python tools/tune.py --around "grid_waves=0,1,2,4" hh_subset >> $O/tune.jsonl 2>> $O/tune.err
