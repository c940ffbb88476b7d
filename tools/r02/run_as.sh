cd $GRAFT_REPO_ROOT
O=gpurun_out/r02as
mkdir -p $O
timeout 800 python tools/e2e_phases.py > $O/phases2.json 2> $O/phases2.err
timeout 1500 python -m pytest tests/test_gpu_column.py -q -p no:cacheprovider -x > $O/gputests.log 2>&1; echo "rc=$?" >> $O/gputests.log
timeout 900 python bench.py --workload column --no-cpu --no-sustained > $O/col.json 2> $O/col.err
