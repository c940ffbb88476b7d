cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -k "relaxed" 2>&1 | tail -3 > gpurun_out/quot_tests.log
TUNE_WARMUP=50 timeout 600 python tools/tune.py --around "recip=1 quot=0,1 fast_path=1" K_Pst SKv3_1 > gpurun_out/tune_quot.jsonl 2> gpurun_out/tune_quot.err
cat gpurun_out/quot_tests.log
