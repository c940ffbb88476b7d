cd $GRAFT_REPO_ROOT
O=gpurun_out/r02af
mkdir -p $O
timeout 600 python bench.py --workload kinetic1m --no-also --no-e2e --no-cpu --warmup 100 --steps 50 > $O/kin.json 2> $O/kin.err
timeout 600 python bench.py --workload kinetic1m_grouped --no-also --no-e2e --no-cpu --warmup 100 --steps 50 > $O/king.json 2> $O/king.err
