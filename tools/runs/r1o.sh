mkdir -p gpurun_out
T=r1o
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
timeout 600 python bench.py --steps 1 --warmup 1 --skip-cpu > gpurun_out/${T}_plain.log 2>&1 && \
  timeout 900 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "acp_step/" -k regex:"k_qrcp_cluster|k_lu_solve|k_jacobi" -c 3 -f -o gpurun_out/${T}_seq \
    python bench.py --steps 1 --warmup 1 --skip-cpu > gpurun_out/${T}_ncu.log 2>&1
echo "ncu rc $?"; tail -3 gpurun_out/${T}_ncu.log
