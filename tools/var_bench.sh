#!/bin/bash
# developer experiment: bench config 5 phases with alternative builds of the library (PX_LIB)
# usage: tools/var_bench.sh lib1.so lib2.so ...   (first entry "default" = the in-tree library)
for lib in "$@"; do
  if [ "$lib" = default ]; then unset PX_LIB; else export PX_LIB=$PWD/$lib; fi
  python bench.py --steps 4 --warmup 3 --no-cpu-baseline --e2e-steps 0 ${VB_ARGS} > gpurun_out/vb.log 2>&1 || { echo "$lib FAILED"; tail -5 gpurun_out/vb.log; continue; }
  python - "$lib" <<'PY'
import json,sys
d=json.loads(open('gpurun_out/vb.log').read().strip().splitlines()[-1])
p=d['phases']
print(sys.argv[1], 'ms/step %.1f'%d['ms_per_step'], ' '.join('%s=%.1f'%(k,v['ms_per_step']) for k,v in p.items()), 'clk', d['clocks']['sm_mhz'])
PY
done
