mkdir -p gpurun_out
T=${TAG:-R2h}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
timeout 240 python -m pytest tests/test_gpu_parity.py -q -x -k "fused or 2d or three_pass" > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/${T}_pytest.log
for CN in "c3g_2d_8x8 7680" "c4g_2d_16x16 4096"; do
set -- $CN
for E in X=1 ACP_F2C_MB=2 ACP_F2C_OFF=1; do
env ${E%%=*}=${E#*=} timeout 120 python tools/k1_time.py $1 $2 > gpurun_out/${T}_t.log 2>&1; echo "$E $(tail -1 gpurun_out/${T}_t.log | cut -c1-120)"
done; done
