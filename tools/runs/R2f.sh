# Round 2, call f: fused 2D K1 variants (skew), timing only
mkdir -p gpurun_out
T=${TAG:-R2f}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "fused" > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc $?"; tail -1 gpurun_out/${T}_pytest.log
for CN in "c3g_2d_8x8 7680" "c4g_2d_16x16 4096"; do
set -- $CN
for E in X=1 ACP_F2C_SKEW=4 ACP_F2C_SKEW=6 ACP_F2C_SKEW=12 ACP_F2C_OFF=1; do
env ${E%%=*}=${E#*=} timeout 300 python tools/k1_time.py $1 $2 > gpurun_out/${T}_t.log 2>&1; echo "$E $(tail -1 gpurun_out/${T}_t.log | cut -c1-120)"
done; done
