#!/bin/bash
# ncu evidence, round 2. Run under gpurun (one GPU); each ncu command runs only after the
# identical plain command exited 0.
set -x
mkdir -p gpurun_out
CMD="python bench.py --profile-only --warmup 0 --steps 1"
$CMD > gpurun_out/plain_c5.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/r02_launches_c5.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo launches=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_rk4_marchc -s 3 -c 1 -o gpurun_out/r02_prof_marchc_dir_c5 $CMD > gpurun_out/ncu_mcd.log 2>&1
echo marchc_dir=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cheb_march -s 20 -c 3 -o gpurun_out/r02_prof_cheb_c5 $CMD > gpurun_out/ncu_cheb.log 2>&1
echo cheb=$?
HCMD="python tools/hybrid_bench.py"
$HCMD > gpurun_out/plain_hyb.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_hyb_ -c 4 -o gpurun_out/r02_prof_hybrid_c3 $HCMD > gpurun_out/ncu_hyb.log 2>&1
echo hyb=$?
