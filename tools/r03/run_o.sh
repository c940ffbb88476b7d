cd $GRAFT_REPO_ROOT
O=gpurun_out/r03o
mkdir -p $O
i=0
for v in "" "ilp=1" "ilp=1,grid_waves=1" "pipe=0" "ilp=2,grid_waves=1" "ilp=2,min_blocks=3" "ilp=2,block=128,min_blocks=8" ""; do
  i=$((i+1))
  NMODL_OPT_Ih="$v" timeout 300 python bench.py --workload column --cells 12500 --no-e2e --no-cpu --no-sustained > $O/col12k_$i.json 2> $O/col12k_$i.err
  echo "$i $v" >> $O/variants.txt
done
