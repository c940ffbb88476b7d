cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r02b
nproc > gpurun_out/r02b/nproc.txt
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=25 > gpurun_out/r02b/gputests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02b/gputests.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/r02b/smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/r02b/smoke.log
timeout 900 python bench.py > gpurun_out/r02b/bench.json 2> gpurun_out/r02b/bench.err
echo "bench rc=$?" >> gpurun_out/r02b/bench.err
