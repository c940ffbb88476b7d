cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_nodes.py -q -x 2>&1 | tail -15 > gpurun_out/warptiles_tests.log
{
timeout 600 python tools/tune.py --grid "ilp=1 fast_path=0 warp_tiles=1 tile=128,256,384 block=256 min_blocks=0,4" ProbAMPANMDA_EMS
timeout 600 python tools/tune.py --grid "ilp=1 fast_path=0 warp_tiles=1 tile=128,192 block=512 min_blocks=0,2" ProbAMPANMDA_EMS
timeout 300 python tools/tune.py --grid "ilp=1 fast_path=0 tile=2048" ProbAMPANMDA_EMS
} > gpurun_out/tune_warptiles.jsonl 2> gpurun_out/tune_warptiles.err
tail -4 gpurun_out/warptiles_tests.log
