cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_nodes.py -q -x 2>&1 | tail -15 > gpurun_out/nodepipe_tests.log
timeout 900 python tools/tune.py --grid "ilp=1 fast_path=0 pipe=1 tile=1024,2048,4096 min_blocks=0,3,4" ProbAMPANMDA_EMS > gpurun_out/tune_nodepipe.jsonl 2> gpurun_out/tune_nodepipe.err
timeout 900 python tools/tune.py --grid "ilp=1 fast_path=1 fast_redo=1 pipe=1 tile=1024,2048,4096 min_blocks=0,3,4" ProbAMPANMDA_EMS >> gpurun_out/tune_nodepipe.jsonl 2>> gpurun_out/tune_nodepipe.err
timeout 300 python tools/tune.py --grid "ilp=1 fast_path=0 pipe=0 tile=2048" ProbAMPANMDA_EMS >> gpurun_out/tune_nodepipe.jsonl 2>> gpurun_out/tune_nodepipe.err
tail -4 gpurun_out/nodepipe_tests.log
