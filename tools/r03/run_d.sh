cd $GRAFT_REPO_ROOT
O=gpurun_out/r03d
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_column.py tests/test_gpu_nodes.py tests/test_gpu_fullsize.py -k "column or node or unique" -q -p no:cacheprovider -x > $O/gputests.log 2>&1; echo "pytest rc=$?" >> $O/gputests.log
for i in 1 2; do
for p in 1 0; do
NMODL_COMBINE_PDL=$p timeout 300 python bench.py --workload column --cells 12500 --no-e2e --no-cpu --no-sustained > $O/col12k_pdl${p}_$i.json 2> $O/col12k_pdl${p}_$i.err
done
done
NMODL_COMBINE_PDL=1 timeout 600 python bench.py --workload column --no-e2e --no-cpu --no-sustained > $O/col100k_pdl1.json 2> $O/col100k_pdl1.err
NMODL_COMBINE_PDL=0 timeout 600 python bench.py --workload column --no-e2e --no-cpu --no-sustained > $O/col100k_pdl0.json 2> $O/col100k_pdl0.err
