#!/bin/bash
# Round-end evidence in one gpurun call, outputs kept under 64 MiB:
# tests + every bench config (final_run.sh), then per config the ncu launch
# list, the 8-launch DRAM capture and one --set full capture, summarised on
# the box (the .ncu-rep and the source page are deleted after summarising).
T=${1:-r02s3f}
bash tools/final_run.sh $T
ALGO_c2=50331648; ALGO_c3=201326592; ALGO_c4=402653184; ALGO_c5=12884901888; ALGO_large=50331648
for c in c2 c3 c4 c5 large; do
  k=lean_kernel; [ $c = large ] && k=batch_kernel
  timeout 900 bash tools/ncu_c2.sh $c $T $k
  a=ALGO_$c
  python tools/ncu_summary.py gpurun_out/${T}_${c}_raw.csv gpurun_out/${T}_${c}_step ${!a} > /dev/null 2>&1
  python tools/ncu_phases.py gpurun_out/${T}_${c}_source.csv > gpurun_out/${T}_${c}_phases.txt 2>&1
  rm -f gpurun_out/${T}_${c}.ncu-rep gpurun_out/${T}_${c}_source.csv
done
du -sh gpurun_out
ls gpurun_out | grep $T
tail -3 gpurun_out/${T}_gputest.log
