#!/bin/bash
# K1 (fused 2D k_f2c) batches-per-item x queue-skew A/B at c4g's production width, same box.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/R5g_build.log 2>&1 || { tail -20 gpurun_out/R5g_build.log; exit 1; }
P=paper_1605_08021_b200
cp $P/libacp_b200.so /tmp/lib_default.so
FL="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr"
run() { for s in $2; do ACP_F2C_SKEW=$s timeout 300 python tools/k1_time.py c4g_2d_16x16 38088 10 0 2>&1 | grep '^{' | sed "s/^{/{\"bpi\": \"$1\", /"; done; }
run 2 "16" > gpurun_out/R5g_k1.txt
for v in 4 8 16; do
  nvcc $FL -DACP_F2C_BPI=$v -c $P/csrc/fft2c.cu -o $P/build/fft2c.o && \
  nvcc -shared -gencode arch=compute_100a,code=sm_100a $P/build/*.o -o $P/libacp_b200.so -lcudart && \
  case $v in 4) run 4 "12 16 20 28 36" ;; 8) run 8 "12 16 24 32 52" ;; 16) run 16 "12 16 24 32 48" ;; esac >> gpurun_out/R5g_k1.txt
done
cp /tmp/lib_default.so $P/libacp_b200.so
run 2 "16" >> gpurun_out/R5g_k1.txt
python - <<'PY'
import json
for l in open("gpurun_out/R5g_k1.txt"):
    d=json.loads(l); print(d["bpi"], d["env"].get("ACP_F2C_SKEW"), round(d["us"]/1e3,3))
PY
