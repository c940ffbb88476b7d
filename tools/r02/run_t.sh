cd $GRAFT_REPO_ROOT
O=gpurun_out/r02t
mkdir -p $O
for pdl in 0 1; do
export NMODL_PDL=$pdl
for cells in 100000 12500; do
timeout 600 python bench.py --workload column --cells $cells --no-e2e --no-cpu --no-sustained > $O/col_${cells}_pdl$pdl.json 2> $O/col_${cells}_pdl$pdl.err
done
timeout 900 python bench.py --no-e2e --no-cpu --no-sustained > $O/bench_pdl$pdl.json 2> $O/bench_pdl$pdl.err
done
