set -x
timeout 2400 python tests/fuzz_campaign.py 10000 14000 > gpurun_out/r02_fuzz_campaign.txt 2>&1; echo rc=$?
tail -3 gpurun_out/r02_fuzz_campaign.txt
timeout 900 python -m paper_1710_08332_b200.cli fuzz --device cuda --junit gpurun_out/r02_fuzz_junit.xml > gpurun_out/r02_cli_fuzz.txt 2>&1; echo rc=$?
head -3 gpurun_out/r02_cli_fuzz.txt
