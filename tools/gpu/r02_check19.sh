set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -8
python __graft_entry__.py smoke; echo smoke rc=$?
start=$(date +%s); timeout 1200 python bench.py > gpurun_out/c19_bench.json 2> gpurun_out/c19_bench.err; echo "bench rc=$? wall=$(( $(date +%s) - start ))s"
tail -c 600 gpurun_out/c19_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/c19_ref.json 2> gpurun_out/c19_ref.err; echo ref rc=$?
python - <<'PY'
import json
d = json.loads(open("gpurun_out/c19_bench.json").read().strip().splitlines()[-1])
print(d["value"], d["roofline"]["frac"], d["roofline"]["isolated"]["frac"], d["e2e"]["value"], d["clocks"])
for k, v in d["suite"].items():
    r = v["roofline"]
    print("  ", k, v["value"], r["frac"], r.get("isolated", {}).get("frac"), r.get("frac_of_size_matched_sol"), r.get("traffic_over_algorithmic"))
PY
