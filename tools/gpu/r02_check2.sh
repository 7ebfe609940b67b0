set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -15
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/c2_b1.json 2> gpurun_out/c2_b1.err; echo rc=$?
timeout 300 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/c2_ref.json 2> gpurun_out/c2_ref.err; echo rc=$?
python __graft_entry__.py smoke
