cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_parity.py -k "relaxed or faithful" -q 2>&1 | tail -15 > gpurun_out/exp16_tests.log
timeout 900 python tools/tune.py --around "exp_smem=0,1 fast_path=0,1" hh_subset NaTs2_t K_Pst Ca_HVA SKv3_1 Ih na6 cdp5ish cadyn ProbAMPANMDA_EMS > gpurun_out/tune_exp16.jsonl 2> gpurun_out/tune_exp16.err
cat gpurun_out/exp16_tests.log | tail -5
