cd $GRAFT_REPO_ROOT
O=gpurun_out/r02ah
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_nodes.py -q -p no:cacheprovider -k "window" > $O/gputests.log 2>&1; echo "rc=$?" >> $O/gputests.log
export TUNE_WARMUP=30
timeout 900 python tools/tune.py --around "vwin=0,1" ProbAMPANMDA_EMS > $O/tune_vwin.jsonl 2> $O/tune.err
TUNE_N=1250000 TUNE_NODES=262500 timeout 900 python tools/tune.py --around "vwin=0,1" ProbAMPANMDA_EMS >> $O/tune_vwin.jsonl 2>> $O/tune.err
