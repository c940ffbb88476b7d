set -x
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py -k cp_async -x -q 2>&1 | tail -5 > gpurun_out/pipe_tests.log
T="timeout 300 python tools/tune.py"
{
$T --grid "ilp=1,2 fast_path=0,1 min_blocks=0,4 pipe=0,1" hh_subset
$T --grid "ilp=1,2 fast_path=0,1 pipe=0,1" NaTs2_t K_Pst Ca_HVA na6 cdp5ish
$T --grid "ilp=1,2 pipe=0,1" SKv3_1 Ih cadyn
$T --grid "ilp=1,2 fast_path=1 min_blocks=2 pipe=0,1" na6 cdp5ish NaTs2_t
} > gpurun_out/tune_pipe.jsonl 2> gpurun_out/tune_pipe.err
cat gpurun_out/pipe_tests.log
