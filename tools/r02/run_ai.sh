cd $GRAFT_REPO_ROOT
O=gpurun_out/r02ai
mkdir -p $O
for v in "" "min_blocks=4"; do
tag=${v:-base}
export NMODL_OPT_Ih="$v"
[ -z "$v" ] && unset NMODL_OPT_Ih
for cells in 100000 12500; do
timeout 600 python bench.py --workload column --cells $cells --no-e2e --no-cpu > $O/col_${cells}_$tag.json 2> $O/col_${cells}_$tag.err
done
timeout 600 python bench.py --workload bbp20m --no-also --no-e2e --no-cpu > $O/bbp_$tag.json 2> $O/bbp_$tag.err
done
