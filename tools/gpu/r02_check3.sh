set -x
python tools/dotbound.py > gpurun_out/dotbound.txt 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv python tools/dotbound.py --ncu > gpurun_out/dotbound_ncu.csv 2> gpurun_out/dotbound_ncu.err
python tools/litgeo.py > gpurun_out/litgeo.txt 2>&1
time (python bench.py --steps 10 --warmup 3 --no-suite > gpurun_out/c3_b1.json 2> gpurun_out/c3_b1.err)
cat gpurun_out/dotbound.txt gpurun_out/litgeo.txt
