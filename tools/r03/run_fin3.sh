cd $GRAFT_REPO_ROOT
O=gpurun_out/r03fin3
mkdir -p $O
nproc > $O/nproc.txt
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rs --durations=10 > $O/gputests.log 2>&1; echo "pytest rc=$?" >> $O/gputests.log
timeout 300 python __graft_entry__.py smoke > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
export PROFILE_TAG=r03fin3_prof
timeout 1500 python tools/profile_bench.py $O/prof > $O/profile.log 2>&1; echo "rc=$?" >> $O/profile.log
rm -f $O/prof/*.ncu-rep
NMODL_COLUMN_CELLS=12500 PROFILE_TAG=r03fin3_prof12k timeout 900 python tools/profile_bench.py $O/prof12k column > $O/prof12k.log 2>&1; echo "rc=$?" >> $O/prof12k.log
rm -f $O/prof12k/*.ncu-rep
python - <<'PY'
import json
a = json.load(open("profiles/ncu_traffic.json"))
for src in ("gpurun_out/r03fin3/prof/ncu_traffic.json", "gpurun_out/r03fin3/prof12k/ncu_traffic.json"):
    try:
        a["by_build"].update(json.load(open(src))["by_build"])
    except Exception as exc:
        print("merge", src, exc)
json.dump(a, open("profiles/ncu_traffic.json", "w"), indent=1, sort_keys=True)
json.dump(a, open("gpurun_out/r03fin3/ncu_traffic_merged.json", "w"), indent=1, sort_keys=True)
PY
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
timeout 600 python bench.py --workload column > $O/bench_column.json 2> $O/bench_column.err; echo "rc=$?" >> $O/bench_column.err
timeout 600 python bench.py --workload column --cells 12500 --no-e2e --no-cpu > $O/bench_column_12500.json 2> $O/bench_column_12500.err
timeout 600 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 20 --warmup 3 --no-also --no-e2e > $O/bench_n2.json 2> $O/bench_n2.err; echo "rc=$?" >> $O/bench_n2.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_synapse.csv python bench.py --steps 20 --warmup 5 --no-also --no-e2e --no-cpu --no-sustained > $O/ncu_bench.log 2>&1
