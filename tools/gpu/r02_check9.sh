set -x
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_reference_parity.py tests/test_gpu_refast.py tests/test_sanitizer.py tests/test_strategy_fuzz.py tests/test_shard.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -5
python tools/litgeo.py --quick 2>&1 | tee gpurun_out/r02_litgeo_vec.txt
python bench.py --workload dot_literal --no-suite --no-cpu --steps 20 --warmup 5 > gpurun_out/c9_lit.json 2>&1
tail -c 600 gpurun_out/c9_lit.json
