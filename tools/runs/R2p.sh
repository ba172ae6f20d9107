mkdir -p gpurun_out
T=${TAG:-R2p}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
for C in c2_1d_semiconductor c3g_2d_8x8 c4g_2d_16x16; do
ACP_QRCP_KRON=1 timeout 300 python tools/qr_time.py $C 1 > gpurun_out/${T}_q.log 2>&1; tail -1 gpurun_out/${T}_q.log | cut -c1-110
ACP_KQ_PROF=1 ACP_QRCP_KRON=1 timeout 300 python tools/qr_time.py $C 1 2>&1 | grep kq | tail -1
done
