cd $GRAFT_REPO_ROOT
P="ncu --set full --clock-control none --import-source on"
$P -k regex:ProbAMPANMDA_EMS_k_step_nodes -s 5 -c 1 -o gpurun_out/r1j_synapse -f python bench.py --steps 3 --warmup 3 --no-also --no-e2e > gpurun_out/r1j_syn.log 2>&1
$P -s 3 -c 1 -k regex:hh_k_step -o gpurun_out/r1j_hh -f python tools/prof_variant.py hh_subset 1000000 ilp=1 fast_path=True pipe=True recip=True div_approx=True exp_share=True fast_redo=True > gpurun_out/r1j_hh.log 2>&1
$P -s 3 -c 1 -k regex:NaTs2_t_k_step -o gpurun_out/r1j_NaTs2_t -f python tools/prof_variant.py NaTs2_t 3333333 ilp=2 min_blocks=2 fast_path=True pipe=True recip=True div_approx=True exp_share=True fast_redo=True > gpurun_out/r1j_nats.log 2>&1
$P -s 3 -c 1 -k regex:K_Pst_k_step -o gpurun_out/r1j_K_Pst -f python tools/prof_variant.py K_Pst 3333333 ilp=2 min_blocks=2 fast_path=True pipe=True recip=True quot=True div_approx=True exp_smem=True exp_share=True fast_redo=True > gpurun_out/r1j_kpst.log 2>&1
ls gpurun_out/r1j*.ncu-rep
