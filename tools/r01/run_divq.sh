cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "relaxed or fallback" 2>&1 | tail -4 > gpurun_out/divq_tests.log
TUNE_WARMUP=150 timeout 600 python tools/tune.py --around "fast_path=1" hh_subset NaTs2_t K_Pst SKv3_1 cdp5ish Ca_HVA Ih na6 > gpurun_out/tune_divq.jsonl 2> gpurun_out/tune_divq.err
cat gpurun_out/divq_tests.log
