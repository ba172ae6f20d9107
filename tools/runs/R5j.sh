#!/bin/bash
# Kronecker QRCP (c4g compress): L2 policy for the per-pivot Psi pass (share of grid points pinned
# evict_last, rest evict_first) and for the Q passes.  Same box.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/R5j_build.log 2>&1 || { tail -20 gpurun_out/R5j_build.log; exit 1; }
for v in "-1 0" "0 0" "30 0" "50 0" "70 0" "90 0" "-1 1" "50 1" "70 1" "-1 0"; do
  set -- $v
  echo "psi_keep=$1 q_last=$2"
  ACP_KQ_PSI_KEEP=$1 ACP_KQ_QLAST=$2 ACP_KQ_PROF=1 timeout 300 python tools/qr_time.py c4g_2d_16x16 3 2>&1 | grep -E "kq CTA0|^\{" | cut -c1-130
done > gpurun_out/R5j_kq_l2.txt
cat gpurun_out/R5j_kq_l2.txt
