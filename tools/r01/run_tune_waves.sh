cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_nodes.py -k "grid_waves or cp_async" -x -q 2>&1 | tail -5 > gpurun_out/waves_tests.log
T="timeout 400 python tools/tune.py"
{
$T --grid "ilp=1 fast_path=1 pipe=0,1 grid_waves=1,0,2,4" hh_subset
$T --grid "ilp=1 fast_path=0 min_blocks=4 pipe=0,1 grid_waves=1,0,2,4" hh_subset
$T --grid "ilp=1,2 fast_path=1 pipe=0,1 grid_waves=1,0,2,4" NaTs2_t K_Pst Ca_HVA na6 cdp5ish SKv3_1 Ih cadyn
$T --grid "ilp=1 fast_path=0 grid_waves=1,0,2,4 tile=2048,1024" ProbAMPANMDA_EMS
} > gpurun_out/tune_waves.jsonl 2> gpurun_out/tune_waves.err
cat gpurun_out/waves_tests.log
