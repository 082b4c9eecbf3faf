#!/bin/bash
# ncu evidence for one bench config (default c2), run on the GPU box from the
# repo root after `python bench.py --config $CFG` exited 0 without ncu:
#   1. launch list (--metrics gpu__time_duration.sum, every kernel, cold)
#   2. DRAM bytes per launch over 8 CONSECUTIVE ring-rotated step launches
#      with --cache-control none: the previous launches' frames are evicted
#      from L2 during each launch, so dram__bytes_write reaches the steady
#      state (~ the 50.3 MB of frames at c2) instead of the L2-resident
#      single-launch figure
#   3. one --set full capture of a step launch with source / SASS lines
# Outputs under gpurun_out/ (TAG prefix).
CFG=${1:-c2}
TAG=${2:-r02}
# the step kernel: one-wave batches (c2) launch lean_kernel, multi-wave ones
# batch_kernel (whose reset launch comes first: skip it)
KRN=${3:-lean_kernel}
mkdir -p gpurun_out
B="python bench.py --config $CFG --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 5"
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/${TAG}_launches_${CFG}.csv $B > gpurun_out/${TAG}_ncu_launch.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_write.sum,dram__bytes_read.sum,lts__t_bytes.sum \
  --cache-control none --clock-control none -k regex:$KRN --launch-skip 3 -c 8 --csv \
  --log-file gpurun_out/${TAG}_dram8_${CFG}.csv $B > gpurun_out/${TAG}_ncu_dram.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:$KRN --launch-skip 6 -c 1 \
  -f -o gpurun_out/${TAG}_${CFG} $B > gpurun_out/${TAG}_ncu_full.log 2>&1
ncu -i gpurun_out/${TAG}_${CFG}.ncu-rep --page source --csv --print-source cuda,sass \
  > gpurun_out/${TAG}_${CFG}_source.csv 2>/dev/null
ncu -i gpurun_out/${TAG}_${CFG}.ncu-rep --page raw --csv > gpurun_out/${TAG}_${CFG}_raw.csv 2>/dev/null
