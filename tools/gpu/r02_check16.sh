set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
start=$(date +%s); timeout 1200 python bench.py > gpurun_out/c16_bench.json 2> gpurun_out/c16_bench.err; echo "bench rc=$? wall=$(( $(date +%s) - start ))s"
tail -c 600 gpurun_out/c16_bench.err
DPIA_BENCH_SHARE_GPU=1 timeout 900 python bench.py --gpus 2 --steps 10 > gpurun_out/c16_w2.json 2> gpurun_out/c16_w2.err; echo w2 rc=$?
tail -c 600 gpurun_out/c16_w2.err
python - <<'PY'
import json
for f in ("gpurun_out/c16_bench.json", "gpurun_out/c16_w2.json"):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "unreadable", e); continue
    print(f, d["value"], d["roofline"]["frac"], d["roofline"].get("isolated"), d["config"].get("input_sets"))
    for k, v in d["suite"].items():
        r = v["roofline"]
        print("  ", k, v["value"], r["frac"], r.get("isolated", {}).get("frac"), v["config"].get("input_sets"))
PY
