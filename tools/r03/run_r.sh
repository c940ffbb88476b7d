cd $GRAFT_REPO_ROOT
O=gpurun_out/r03r
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -rs > $O/gputests.log 2>&1; echo "pytest rc=$?" >> $O/gputests.log
PROFILE_TAG=r03fin2_prof timeout 1500 python tools/profile_bench.py $O/prof kinetic1m kinetic10m kinetic1m_grouped > $O/profile.log 2>&1; echo "rc=$?" >> $O/profile.log
rm -f $O/prof/*.ncu-rep
python - <<'PY'
import json
a = json.load(open("profiles/ncu_traffic.json"))
a["by_build"].update(json.load(open("gpurun_out/r03r/prof/ncu_traffic.json"))["by_build"])
json.dump(a, open("profiles/ncu_traffic.json", "w"), indent=1, sort_keys=True)
json.dump(a, open("gpurun_out/r03r/ncu_traffic_merged.json", "w"), indent=1, sort_keys=True)
PY
for i in 1 2; do
timeout 600 python bench.py > $O/bench_$i.json 2> $O/bench_$i.err
done
