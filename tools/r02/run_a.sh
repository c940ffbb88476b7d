cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r02a
./tools/micro/flush_modes > gpurun_out/r02a/flush_modes.jsonl 2>&1
TUNE_WARMUP=50 timeout 900 python tools/tune.py --around "block=128 min_blocks=0,4,5,6" hh_subset K_Pst NaTs2_t > gpurun_out/r02a/tune_block128.jsonl 2> gpurun_out/r02a/tune.err
TUNE_WARMUP=50 timeout 600 python tools/tune.py --around "block=64 min_blocks=0,8,10,12" hh_subset K_Pst >> gpurun_out/r02a/tune_block64.jsonl 2>> gpurun_out/r02a/tune.err
TUNE_N=10000000 TUNE_WARMUP=20 timeout 300 python tools/tune.py --around "block=256" hh_subset > gpurun_out/r02a/tune_hh10m.jsonl 2>> gpurun_out/r02a/tune.err
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv >> gpurun_out/r02a/smi.txt
