cd $GRAFT_REPO_ROOT
timeout 600 python bench.py --workload column --steps 50 --warmup 5 > gpurun_out/bench_column.json 2> gpurun_out/bench_column.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r1i_synapse.csv python bench.py --steps 20 --warmup 5 --no-also --no-e2e > gpurun_out/ncu_bench.log 2>&1
P="ncu --set full --clock-control none --import-source on -s 3 -c 1"
$P -k regex:K_Pst_k_step -o gpurun_out/r1i_K_Pst -f python tools/prof_variant.py K_Pst 3333333 ilp=2 min_blocks=2 fast_path=True pipe=True div_approx=True fast_redo=True > gpurun_out/r1i_kpst.log 2>&1
$P -k regex:na6_k_step -o gpurun_out/r1i_na6 -f python tools/prof_variant.py na6 1000000 ilp=1 min_blocks=2 fast_path=True pipe=True fast_redo=True lu_spec=True > gpurun_out/r1i_na6.log 2>&1
$P -k regex:cdp5ish_k_step -o gpurun_out/r1i_cdp5ish -f python tools/prof_variant.py cdp5ish 1000000 ilp=1 min_blocks=2 fast_path=True pipe=True div_approx=True fast_redo=True lu_spec=True > gpurun_out/r1i_cdp5.log 2>&1
$P -k regex:hh_k_step -o gpurun_out/r1i_hh -f python tools/prof_variant.py hh_subset 1000000 ilp=1 fast_path=True pipe=True recip=True div_approx=True fast_redo=True > gpurun_out/r1i_hh.log 2>&1
$P -k regex:NaTs2_t_k_step -o gpurun_out/r1i_NaTs2_t -f python tools/prof_variant.py NaTs2_t 3333333 ilp=2 min_blocks=2 fast_path=True pipe=True recip=True div_approx=True fast_redo=True > gpurun_out/r1i_nats.log 2>&1
ls gpurun_out/*.ncu-rep; cat gpurun_out/bench_ref.json | head -c 600
