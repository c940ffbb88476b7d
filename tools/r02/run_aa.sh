cd $GRAFT_REPO_ROOT
O=gpurun_out/r02aa
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_nodes.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -p no:cacheprovider -x > $O/gputests.log 2>&1; echo "pytest rc=$?" >> $O/gputests.log
timeout 900 python bench.py --no-also --no-cpu --no-sustained > $O/bench.json 2> $O/bench.err
