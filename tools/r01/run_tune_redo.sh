cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_parity.py -k "fallback or relaxed" -q 2>&1 | tail -15 > gpurun_out/redo_tests.log
timeout 900 python tools/tune.py --around "fast_redo=0,1 min_blocks=0,2,3 fast_path=1" hh_subset NaTs2_t K_Pst Ca_HVA SKv3_1 Ih na6 cdp5ish ProbAMPANMDA_EMS > gpurun_out/tune_redo.jsonl 2> gpurun_out/tune_redo.err
tail -5 gpurun_out/redo_tests.log
