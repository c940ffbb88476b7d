cd $GRAFT_REPO_ROOT
O=gpurun_out/r02ac
mkdir -p $O
timeout 900 python tools/stream_pdl.py > $O/stream_pdl.jsonl 2> $O/err.txt
