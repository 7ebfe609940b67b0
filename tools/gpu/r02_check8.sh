python tools/litexp.py 2>&1 | tee gpurun_out/r02_litexp.txt
