mkdir -p gpurun_out
T=r2t
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
ACP_F2_CB16=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "fourier and 2d" > gpurun_out/${T}_pytest.log 2>&1; echo "pytest cb16 rc $?"; tail -1 gpurun_out/${T}_pytest.log
for K in X ACP_F2_CB16 X ACP_F2_CB16; do
echo "$K c3g $(env $K=1 timeout 300 python tools/k1_sweep.py c3g_2d_8x8 6688 2>&1 | tail -1)"
echo "$K c4g $(env $K=1 timeout 300 python tools/k1_sweep.py c4g_2d_16x16 4096 2>&1 | tail -1)"
done
