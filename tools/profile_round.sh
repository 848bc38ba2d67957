#!/bin/bash
# Round-end evidence (run under gpurun, 1 GPU).  Outputs land in gpurun_out/;
# tools/summarize_ncu.py and tools/lttb_table.py turn them into profiles/<tag>_*.
TAG=${1:-r01}
python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
python tools/configs_time.py > gpurun_out/${TAG}_configs.md 2> gpurun_out/${TAG}_configs.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 5 --warmup 3 --no-cpu \
    > gpurun_out/${TAG}_ncu_launches.log 2>&1
python tools/profile_scan.py c2 3 > gpurun_out/${TAG}_plain_c2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:scan_kernel -s 1 -c 1 \
    -o gpurun_out/${TAG}_scan_c2 -f python tools/profile_scan.py c2 3 > gpurun_out/${TAG}_ncu_full.log 2>&1
for n in 1000 10000; do
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      --cache-control none --csv --log-file gpurun_out/${TAG}_lttb_launches_$n.csv \
      python tools/profile_lttb.py $n 2 > gpurun_out/${TAG}_ncu_lttb_$n.log 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:lttb_sb_kernel -s 1 -c 1 \
    -o gpurun_out/${TAG}_lttb_sb -f python tools/profile_lttb.py 1000 2 > gpurun_out/${TAG}_ncu_lttb_sb.log 2>&1

# summarise on the box (ncu -i), keep the summaries, drop the large reports
mkdir -p gpurun_out/prof_${TAG}
PROF_DIR=gpurun_out/prof_${TAG} python tools/summarize_ncu.py ${TAG} > /dev/null 2>&1
ncu -i gpurun_out/${TAG}_lttb_sb.ncu-rep --page details --csv > gpurun_out/prof_${TAG}/${TAG}_lttb_sb_details.csv 2>/dev/null
rm -f gpurun_out/*.ncu-rep
echo summarised
