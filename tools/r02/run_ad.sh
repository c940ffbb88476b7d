cd $GRAFT_REPO_ROOT
O=gpurun_out/r02ad
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_column.py -q -p no:cacheprovider -k "direct_population" > $O/gputests.log 2>&1; echo "rc=$?" >> $O/gputests.log
for g in 0 1; do
NMODL_BBP_GROUPED=$g timeout 600 python bench.py --workload bbp20m --no-also --no-e2e --no-cpu > $O/bbp_g$g.json 2> $O/bbp_g$g.err
done
