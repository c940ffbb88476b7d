cd $GRAFT_REPO_ROOT
O=gpurun_out/r03b
mkdir -p $O
for v in "block=288,min_blocks=4" "block=224,min_blocks=5" "block=192,min_blocks=6" "block=320,min_blocks=3" "block=256,min_blocks=4"; do
  t=$(echo $v | tr ',=' '__')
  NMODL_OPT_ProbAMPANMDA_EMS="$v" timeout 300 python bench.py --workload column --cells 12500 --no-e2e --no-cpu --no-sustained > $O/col12k_$t.json 2> $O/col12k_$t.err
  NMODL_OPT_ProbAMPANMDA_EMS="$v" timeout 300 python bench.py --no-also --no-e2e --no-cpu --no-sustained > $O/syn10m_$t.json 2> $O/syn10m_$t.err
done
