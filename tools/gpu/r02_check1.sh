set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests/test_gpu_reference_parity.py -q -m gpu 2>&1 | tail -25
python -m pytest tests/test_scaleout.py tests/test_shard.py -m gpu -q 2>&1 | tail -5
python -m pytest tests/test_gpu_parity.py -k "fuzz_programs_fp32 or empty or executable_run" -q 2>&1 | tail -5
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/b1.json 2> gpurun_out/b1.err; echo rc=$?
DPIA_BENCH_SHARE_GPU=1 timeout 600 python bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/b2.json 2> gpurun_out/b2.err; echo rc=$?
tail -5 gpurun_out/b2.err
