set -x
timeout 900 python tools/litpf.py > gpurun_out/r02_litpf2.txt 2>&1; echo litpf rc=$?
cat gpurun_out/r02_litpf2.txt
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_reference_parity.py tests/test_gpu_refast.py tests/test_strategy_fuzz.py tests/test_sanitizer.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -4
