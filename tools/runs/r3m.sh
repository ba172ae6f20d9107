mkdir -p gpurun_out
T=r3m
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "qrcp or compress" > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc $?"; tail -1 gpurun_out/${T}_pytest.log
ACP_QRCP_CHUNK1=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "alternative_qrcp" > gpurun_out/${T}_pytest1.log 2>&1; echo "pytest chunk1 rc $?"; tail -1 gpurun_out/${T}_pytest1.log
for K in X ACP_QRCP_CHUNK1; do
env $K=1 timeout 1500 python bench.py --config c4g_2d_16x16 --steps 1 --warmup 1 --skip-cpu > gpurun_out/${T}_bench_$K.log 2>&1; echo "bench c4g $K rc $? $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/${T}_bench_$K.log | head -1)"
done
