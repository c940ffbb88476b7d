cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_nodes.py -q -x 2>&1 | tail -3 > gpurun_out/idxa_tests.log
{
timeout 600 python tools/tune.py --grid "ilp=1 fast_path=0 idx_ahead=1 tile=1536,2048,3072 min_blocks=0,4" ProbAMPANMDA_EMS
timeout 300 python tools/tune.py --grid "ilp=1 fast_path=0 tile=2048" ProbAMPANMDA_EMS
} > gpurun_out/tune_idxa.jsonl 2> gpurun_out/tune_idxa.err
cat gpurun_out/idxa_tests.log
