set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -6
start=$(date +%s); timeout 1200 python bench.py > gpurun_out/c6_bench.json 2> gpurun_out/c6_bench.err; echo "bench rc=$? wall=$(( $(date +%s) - start ))s"
timeout 600 python bench.py --impl reference > gpurun_out/c6_ref.json 2> gpurun_out/c6_ref.err; echo rc=$?
DPIA_BENCH_SHARE_GPU=1 timeout 900 python bench.py --gpus 2 > gpurun_out/c6_w2.json 2> gpurun_out/c6_w2.err; echo rc=$?
DPIA_BENCH_SHARE_GPU=1 timeout 900 python bench.py --gpus 4 --steps 10 > gpurun_out/c6_w4.json 2> gpurun_out/c6_w4.err; echo rc=$?
timeout 1800 bash tools/profile.sh > gpurun_out/c6_profile.log 2>&1; echo profile rc=$?
python __graft_entry__.py smoke
