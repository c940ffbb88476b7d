cd $GRAFT_REPO_ROOT
O=gpurun_out/r02ak
mkdir -p $O
for i in 1 2; do
timeout 600 python bench.py --workload bbp20m_grouped --no-also --no-e2e --no-cpu --no-sustained > $O/bbpg_$i.json 2> $O/bbpg_$i.err
done
NMODL_OPT_Ih="min_blocks=0" timeout 600 python bench.py --workload bbp20m_grouped --no-also --no-e2e --no-cpu --no-sustained > $O/bbpg_ih0.json 2> $O/bbpg_ih0.err
