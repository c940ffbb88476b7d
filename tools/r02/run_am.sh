cd $GRAFT_REPO_ROOT
O=gpurun_out/r02am
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q -p no:cacheprovider -k column --durations=5 > $O/gputests.log 2>&1; echo "rc=$?" >> $O/gputests.log
