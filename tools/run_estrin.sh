cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -k "relaxed or faithful" 2>&1 | tail -3 > gpurun_out/estrin_tests.log
TUNE_WARMUP=100 timeout 900 python tools/tune.py --around "exp_estrin=0,1 exp_smem=0" hh_subset NaTs2_t K_Pst Ca_HVA SKv3_1 Ih na6 cdp5ish ProbAMPANMDA_EMS > gpurun_out/tune_estrin.jsonl 2> gpurun_out/tune_estrin.err
cat gpurun_out/estrin_tests.log
