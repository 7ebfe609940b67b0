set -x
timeout 600 python tools/chunkread.py 2>&1 | tee gpurun_out/r02_chunkread.txt
