cd $GRAFT_REPO_ROOT
O=gpurun_out/r03u
mkdir -p $O
timeout 600 python tools/r03/divc_parity.py > $O/parity.jsonl 2> $O/parity.err
TUNE_N=3333333 timeout 900 python tools/tune.py --around "divc_approx=0,1" K_Pst NaTs2_t Ca_HVA SKv3_1 Ih >> $O/tune.jsonl 2>> $O/tune.err
TUNE_N=3333333 timeout 900 python tools/tune.py --around "divc_approx=0,1" K_Pst NaTs2_t >> $O/tune.jsonl 2>> $O/tune.err
timeout 600 python tools/tune.py --around "divc_approx=0,1" hh_subset >> $O/tune.jsonl 2>> $O/tune.err
