#!/bin/bash
# K1 at c3g (192^2, 7672 columns): three passes vs fused k_f2c at several queue skews; c4g default
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/R5d_build.log 2>&1 || { tail -20 gpurun_out/R5d_build.log; exit 1; }
for rep in 1 2; do
  ACP_F2C=0 timeout 300 python tools/k1_time.py c3g_2d_8x8 7672 20 0 2>&1 | grep '^{'
  for s in 9 14 20 28; do ACP_F2C=1 ACP_F2C_SKEW=$s timeout 300 python tools/k1_time.py c3g_2d_8x8 7672 20 0 2>&1 | grep '^{'; done
  ACP_F2C=1 timeout 300 python tools/k1_time.py c3g_2d_8x8 7672 20 0 2>&1 | grep '^{'
  timeout 300 python tools/k1_time.py c4g_2d_16x16 38088 10 0 2>&1 | grep '^{'
done > gpurun_out/R5d_k1.txt
cat gpurun_out/R5d_k1.txt | cut -c1-200
