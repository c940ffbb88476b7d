cd $GRAFT_REPO_ROOT
O=gpurun_out/r03j
mkdir -p $O
i=0
for v in "" "exp_share=1" "recip=1,exp_share=1" "div_approx=1" "recip=1,exp_share=1,div_approx=1" ""; do
  i=$((i+1))
  NMODL_OPT_ProbAMPANMDA_EMS="$v" timeout 400 python bench.py --no-also --no-cpu > $O/syn_$i.json 2> $O/syn_$i.err
  echo "$i $v" >> $O/variants.txt
done
