#!/bin/bash
# Round evidence (run under gpurun, 1 GPU): for every bench config a plain run, an ncu
# launch list (per-launch duration + DRAM bytes) and one `ncu --set full` capture of the
# config's streaming kernel; tools/summarize_round.py turns them into profiles/<tag>_*.
# usage: bash tools/profile_round.sh r02 [configs...]
TAG=${1:-r02}; shift
KEYS=${@:-C1 C2 C3_1000 C3_10000 C4 C5_i16 C5_u8 C5_f16}
mkdir -p gpurun_out
declare -A KREGEX=( [C1]=tile_bins_kernel [C2]=scan_kernel [C3_1000]=lttb_sb_kernel [C3_10000]=lttb_guess_kernel
                    [C4]=scan_kernel [C5_i16]=lane_bins_kernel [C5_u8]=lane_bins_kernel [C5_f16]=lane_bins_kernel )
for K in $KEYS; do
  python tools/step_profile.py $K --steps 5 --warmup 3 > gpurun_out/${TAG}_plain_$K.log 2>&1 || { echo "plain $K failed"; continue; }
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      --log-file gpurun_out/${TAG}_launches_$K.csv python tools/step_profile.py $K --steps 2 --warmup 1 --flush none \
      > gpurun_out/${TAG}_ncu_launches_$K.log 2>&1
  ncu --set full --clock-control none --import-source on -k regex:${KREGEX[$K]} -s 2 -c 1 \
      -o gpurun_out/${TAG}_full_$K -f python tools/step_profile.py $K --steps 2 --warmup 1 --flush none \
      > gpurun_out/${TAG}_ncu_full_$K.log 2>&1
  echo "$K: $(tail -1 gpurun_out/${TAG}_plain_$K.log)"
done
python tools/summarize_round.py $TAG --on-box > gpurun_out/${TAG}_summarize.log 2>&1
# keep the reports small enough to travel: drop the big ones
du -sh gpurun_out/*.ncu-rep 2>/dev/null | tail -20
find gpurun_out -name '*.ncu-rep' -size +6M ! -name "*_${KEEP_REP:-none}.ncu-rep" -delete
echo profiled
