set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_reference_parity.py tests/test_gpu_refast.py tests/test_strategy_fuzz.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -4
timeout 900 python tools/litpf.py > gpurun_out/r02_litpf.txt 2>&1; echo litpf rc=$?
timeout 600 python tools/bulkread.py > gpurun_out/r02_bulkread.txt 2>&1; echo bulk rc=$?
cat gpurun_out/r02_litpf.txt gpurun_out/r02_bulkread.txt
