cd $GRAFT_REPO_ROOT
P="ncu --set full --clock-control none --import-source on -s 3 -c 1"
$P -k regex:hh_k_step -o gpurun_out/r1h_hh -f python tools/prof_variant.py hh_subset 1000000 ilp=1 fast_path=True pipe=True recip=True div_approx=True > gpurun_out/r1h_hh.log 2>&1
$P -k regex:NaTs2_t_k_step -o gpurun_out/r1h_NaTs2_t -f python tools/prof_variant.py NaTs2_t 3333333 ilp=2 fast_path=True pipe=True recip=True div_approx=True > gpurun_out/r1h_nats.log 2>&1
$P -k regex:na6_k_step -o gpurun_out/r1h_na6 -f python tools/prof_variant.py na6 1000000 ilp=1 fast_path=True pipe=True min_blocks=2 > gpurun_out/r1h_na6.log 2>&1
$P -k regex:cdp5ish_k_step -o gpurun_out/r1h_cdp5ish -f python tools/prof_variant.py cdp5ish 1000000 ilp=1 fast_path=True pipe=True div_approx=True > gpurun_out/r1h_cdp5.log 2>&1
ls -la gpurun_out/*.ncu-rep
