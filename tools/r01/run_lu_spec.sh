cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "speculative" 2>&1 | tail -15 > gpurun_out/luspec_tests.log
TUNE_WARMUP=150 timeout 600 python tools/tune.py --around "lu_spec=0,1 min_blocks=0,2" na6 cdp5ish > gpurun_out/tune_luspec.jsonl 2> gpurun_out/tune_luspec.err
tail -4 gpurun_out/luspec_tests.log
