set -x
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_reference_parity.py tests/test_sanitizer.py tests/test_strategy_fuzz.py tests/test_phase_sim.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -8
for b in 1 0; do DPIA_BULK_STAGE=$b python bench.py --workload gemv --no-suite --no-cpu --traffic committed --steps 50 --warmup 5 > gpurun_out/c4_gemv_bulk$b.json 2>&1; done
python bench.py --workload dot_literal --no-suite --no-cpu --steps 20 --warmup 5 > gpurun_out/c4_lit.json 2>&1
python - <<'PY'
import json
for f in ["gpurun_out/c4_gemv_bulk1.json", "gpurun_out/c4_gemv_bulk0.json", "gpurun_out/c4_lit.json"]:
    d = json.loads(open(f).read().strip().splitlines()[-1])
    print(f, d["value"], d["roofline"]["frac"], d["roofline"]["kernel_ms"], d["roofline"].get("traffic"))
PY
