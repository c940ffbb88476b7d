cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -k "relaxed" 2>&1 | tail -3 > gpurun_out/lr_tests.log
TUNE_WARMUP=100 timeout 600 python tools/tune.py --around "lu_recip=0,1" na6 > gpurun_out/tune_lr.jsonl 2> gpurun_out/tune_lr.err
cat gpurun_out/lr_tests.log
