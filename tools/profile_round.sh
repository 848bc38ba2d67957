#!/bin/bash
# Profile capture for one round (run under gpurun, 1 GPU).  Outputs land in
# gpurun_out/; tools/summarize_ncu.py turns them into profiles/<tag>_*.
set -e
TAG=${1:-r01}
python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/${TAG}_bench_plain.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 5 --warmup 3 --no-cpu \
    > gpurun_out/${TAG}_ncu_launches.log 2>&1
python tools/profile_scan.py c2 3 > gpurun_out/${TAG}_plain_c2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:scan_kernel -s 1 -c 1 \
    -o gpurun_out/${TAG}_scan_c2 -f python tools/profile_scan.py c2 3 > gpurun_out/${TAG}_ncu_full.log 2>&1
echo profile done
