set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -6
python __graft_entry__.py smoke; echo smoke rc=$?
start=$(date +%s); timeout 1200 python bench.py > gpurun_out/c10_bench.json 2> gpurun_out/c10_bench.err; echo "bench rc=$? wall=$(( $(date +%s) - start ))s"
tail -c 400 gpurun_out/c10_bench.err
