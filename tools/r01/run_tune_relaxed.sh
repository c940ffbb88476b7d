cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -k "relaxed" -q 2>&1 | tail -40 > gpurun_out/relaxed_tests.log
T="timeout 400 python tools/tune.py"
{
$T --grid "ilp=1 fast_path=1 pipe=1 recip=0,1 div_approx=0,1" hh_subset cdp5ish
$T --grid "ilp=2 fast_path=1 pipe=1 recip=0,1 div_approx=0,1" NaTs2_t K_Pst Ca_HVA
$T --grid "ilp=1 fast_path=1 pipe=1 recip=0,1 div_approx=0,1 grid_waves=4" SKv3_1
$T --grid "ilp=2 fast_path=1 pipe=1 recip=0,1 div_approx=0,1 grid_waves=4" Ih
$T --grid "ilp=1 fast_path=1 pipe=1 recip=0,1 div_approx=0,1 min_blocks=2" na6
} > gpurun_out/tune_relaxed2.jsonl 2> gpurun_out/tune_relaxed2.err
cat gpurun_out/relaxed_tests.log | tail -8
