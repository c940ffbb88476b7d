cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -k "relaxed" 2>&1 | tail -3 > gpurun_out/xs_tests.log
TUNE_WARMUP=100 timeout 600 python tools/tune.py --around "exp_share=0,1" hh_subset NaTs2_t K_Pst > gpurun_out/tune_xs.jsonl 2> gpurun_out/tune_xs.err
cat gpurun_out/xs_tests.log
