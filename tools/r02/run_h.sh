cd $GRAFT_REPO_ROOT
O=gpurun_out/r02h
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_nodes.py -q -p no:cacheprovider -k chunk > $O/gputests.log 2>&1; echo "pytest rc=$?" >> $O/gputests.log
for c in 1 2 4 8; do
NMODL_E2E_CHUNKS=$c timeout 600 python bench.py --no-also --no-cpu --no-sustained --steps 20 > $O/syn_chunks$c.json 2> $O/syn_chunks$c.err
done
