mkdir -p gpurun_out
T=r4c
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
ACP_QRCP_W3=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "alternative_qrcp" > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc $?"; tail -1 gpurun_out/${T}_pytest.log
for C in c3g_2d_8x8 c2_1d_semiconductor; do
for K in X ACP_QRCP_W3 X ACP_QRCP_W3; do
env $K=1 timeout 1500 python bench.py --config $C --steps 2 --warmup 2 --skip-cpu > gpurun_out/${T}_bench.log 2>&1; echo "$C $K rc $? $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/${T}_bench.log | head -1)"
done; done
