cd $GRAFT_REPO_ROOT
O=gpurun_out/r02spread
mkdir -p $O
for i in 1 2 3; do
t0=$(date +%s)
timeout 900 python bench.py > $O/bench_$i.json 2> $O/bench_$i.err
echo "wall $(( $(date +%s) - t0 )) s" >> $O/bench_$i.err
done
