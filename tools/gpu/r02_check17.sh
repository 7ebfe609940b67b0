set -x
timeout 900 python -m pytest tests/test_gpu_chain.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -15
start=$(date +%s); timeout 1200 python bench.py > gpurun_out/c17_bench.json 2> gpurun_out/c17_bench.err; echo "bench rc=$? wall=$(( $(date +%s) - start ))s"
tail -c 600 gpurun_out/c17_bench.err
timeout 1200 python bench.py --no-chain --no-cpu --traffic committed > gpurun_out/c17_nochain.json 2> gpurun_out/c17_nochain.err; echo nochain rc=$?
python - <<'PY'
import json
for f in ("gpurun_out/c17_bench.json", "gpurun_out/c17_nochain.json"):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "unreadable", e); continue
    print(f, d["value"], d["roofline"]["frac"], d["roofline"]["isolated"]["frac"], d["config"].get("input_sets"))
    for k, v in d["suite"].items():
        r = v["roofline"]
        print("  ", k, v["value"], r["frac"], r.get("isolated", {}).get("frac"), r.get("traffic_over_algorithmic"))
PY
