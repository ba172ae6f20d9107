#!/bin/bash
# K1 (fused 2D k_f2c) batches-per-item A/B at c4g's production width: BPI = 2 (default) vs 1 / 4,
# each a rebuild of fft2c.o + relink, same box.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/R5f_build.log 2>&1 || { tail -20 gpurun_out/R5f_build.log; exit 1; }
P=paper_1605_08021_b200
cp $P/libacp_b200.so /tmp/lib_default.so
FL="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr"
run() { for r in 1 2; do timeout 300 python tools/k1_time.py c4g_2d_16x16 38088 10 0 2>&1 | grep '^{' | sed "s/^{/{\"bpi\": \"$1\", /"; done; }
run 2 > gpurun_out/R5f_k1_bpi.txt
for v in 1 4; do
  nvcc $FL -DACP_F2C_BPI=$v -c $P/csrc/fft2c.cu -o $P/build/fft2c.o && \
  nvcc -shared -gencode arch=compute_100a,code=sm_100a $P/build/*.o -o $P/libacp_b200.so -lcudart && run $v >> gpurun_out/R5f_k1_bpi.txt
done
cp /tmp/lib_default.so $P/libacp_b200.so
run 2 >> gpurun_out/R5f_k1_bpi.txt
cut -c1-140 gpurun_out/R5f_k1_bpi.txt
