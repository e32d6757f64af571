#!/bin/bash
# dev helper: build libparaexp.so with ptxas stats; optional SASS op histogram of a kernel
set -e
cd /root/repo/paper_2004_00546_b200/csrc
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared -cudart static -lcufft -Xlinker -rpath,/usr/local/cuda/lib64 -Xptxas -v -o ../libparaexp.so paraexp_capi.cu 2>&1 | grep -E "error|${1:-k_rk4_march}" -A2 | grep -E "error|Compiling|registers|spill" || true
if [ -n "$2" ]; then
  cuobjdump -sass ../libparaexp.so | awk -v k="$2" '$0 ~ "Function : "k {f=1; next} f && /Function : / {f=0} f' | grep -E "^\s+/\*[0-9a-f]{4}\*/" > /tmp/k.sass
  echo "instructions: $(wc -l < /tmp/k.sass)"
  awk '{print $2}' /tmp/k.sass | sed 's/\..*//;s/@.*//' | sort | uniq -c | sort -rn | head -${3:-12}
fi
