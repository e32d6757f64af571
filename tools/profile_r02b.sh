#!/bin/bash
# ncu evidence, round 2 (final build: Chebyshev CTAs 128 × 3, the 2D two-field Burgers kernels). Run
# under gpurun (one GPU); each ncu command runs only after the identical plain command exited 0.
set -x
mkdir -p gpurun_out
CMD="python bench.py --profile-only --warmup 0 --steps 1"
$CMD > gpurun_out/plain_c5.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/r02b_launches_c5.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo launches=$?
python tools/launch_summary.py gpurun_out/r02b_launches_c5.csv gpurun_out/r02b_c5_launches_summary.csv > gpurun_out/r02b_c5_launches_summary.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cheb_march -s 20 -c 3 -o gpurun_out/r02b_prof_cheb_c5 $CMD > gpurun_out/ncu_cheb.log 2>&1
echo cheb=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_rk4_marchc -s 3 -c 1 -o gpurun_out/r02b_prof_marchc_dir_c5 $CMD > gpurun_out/ncu_mcd.log 2>&1
echo marchc=$?
HCMD="python tools/hybrid2d_bench.py small"
$HCMD > gpurun_out/plain_h2.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_b2s_ -s 6 -c 3 -o gpurun_out/r02b_prof_hybrid2d $HCMD > gpurun_out/ncu_h2.log 2>&1
echo h2=$?
for r in r02b_prof_cheb_c5 r02b_prof_marchc_dir_c5 r02b_prof_hybrid2d; do
  ncu -i gpurun_out/$r.ncu-rep --page raw --csv > gpurun_out/${r}_raw.csv 2>/dev/null
  ncu -i gpurun_out/$r.ncu-rep --page details --csv > gpurun_out/${r}_details.csv 2>/dev/null
done
ls -la gpurun_out | head -40
