cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r02
nproc > gpurun_out/r02/nproc.txt
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider --durations=25 > gpurun_out/r02/gputests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02/gputests.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/r02/smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/r02/smoke.log
