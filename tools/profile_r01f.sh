#!/bin/bash
# ncu evidence for configs 4 (Krylov) and 2 (1D on-chip scan), round 1 (f). Run under gpurun (one
# GPU); each ncu command runs only after the identical plain command exited 0.
set -x
mkdir -p gpurun_out
for c in 4 2; do
  CMD="python bench.py --config $c --profile-only --warmup 0 --steps 1"
  $CMD > gpurun_out/plain_c$c.log 2>&1 || exit 1
  ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv --log-file gpurun_out/launches_c$c.csv $CMD > gpurun_out/ncu_launch_c$c.log 2>&1
  echo launches_c$c=$?
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_kr_update -s 200 -c 2 -o gpurun_out/prof_kr_update_c4 python bench.py --config 4 --profile-only --warmup 0 --steps 1 > gpurun_out/ncu_kr.log 2>&1
echo kr=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_scan1d -c 2 -o gpurun_out/prof_scan1d_c2 python bench.py --config 2 --profile-only --warmup 0 --steps 1 > gpurun_out/ncu_s1.log 2>&1
echo s1=$?
