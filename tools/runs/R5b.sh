#!/bin/bash
# K1 (fused 2D k_f2c) queue-skew / ring-size A/B at c4g's production width, one box.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/R5b_build.log 2>&1 || { tail -20 gpurun_out/R5b_build.log; exit 1; }
for rep in 1 2; do
for s in ${SKEWS:-9 12}; do
  ACP_F2C_SKEW=$s timeout 300 python tools/k1_time.py c4g_2d_16x16 38088 10 0 2>&1 | grep '^{' | cut -c1-200
done
done > gpurun_out/R5b_k1_skew.txt
cat gpurun_out/R5b_k1_skew.txt
