#!/bin/bash
# Fused 2D K1 with 4 batches per item (new default): parity subset, c4g timing, c3g fused vs three passes.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/R5h_build.log 2>&1 || { tail -20 gpurun_out/R5h_build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "fourier or fused or inactive_pairs or free_electron or tiny2d or c4g_outer0" > gpurun_out/R5h_pytest.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/R5h_pytest.log
for r in 1 2; do
  timeout 300 python tools/k1_time.py c4g_2d_16x16 38088 10 0 2>&1 | grep '^{'
  ACP_F2C=0 timeout 300 python tools/k1_time.py c3g_2d_8x8 7672 20 0 2>&1 | grep '^{'
  for s in 0 12 16 24; do
    if [ $s = 0 ]; then ACP_F2C=1 timeout 300 python tools/k1_time.py c3g_2d_8x8 7672 20 0 2>&1 | grep '^{';
    else ACP_F2C=1 ACP_F2C_SKEW=$s timeout 300 python tools/k1_time.py c3g_2d_8x8 7672 20 0 2>&1 | grep '^{'; fi
  done
done > gpurun_out/R5h_k1.txt
cut -c1-170 gpurun_out/R5h_k1.txt
