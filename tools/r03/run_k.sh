cd $GRAFT_REPO_ROOT
O=gpurun_out/r03k
mkdir -p $O
for i in 1 2 3; do
  timeout 600 python bench.py --no-cpu > $O/bench_$i.json 2> $O/bench_$i.err
  timeout 300 python bench.py --workload column --cells 12500 --no-e2e --no-cpu --no-sustained > $O/col12k_$i.json 2> $O/col12k_$i.err
done
