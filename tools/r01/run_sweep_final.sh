cd $GRAFT_REPO_ROOT
TUNE_WARMUP=100 timeout 1500 python tools/tune.py --around "ilp=1,2 min_blocks=0,2,3 grid_waves=1,4 fast_path=1" hh_subset NaTs2_t K_Pst Ca_HVA SKv3_1 Ih na6 cdp5ish cadyn > gpurun_out/tune_final.jsonl 2> gpurun_out/tune_final.err
