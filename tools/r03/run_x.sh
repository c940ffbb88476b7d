cd $GRAFT_REPO_ROOT
O=gpurun_out/r03x
mkdir -p $O
for n in 1000000 10000000; do
TUNE_N=$n timeout 900 python tools/tune.py --around "recip=0,1 quot=0,1 exp_share=0,1" cdp5ish >> $O/tune.jsonl 2>> $O/tune.err
done
