mkdir -p gpurun_out
T=r1zw
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
timeout 900 python -m pytest tests -q -m gpu -x -k "qrcp or compress" > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc $?"; tail -2 gpurun_out/${T}_pytest.log
for C in c2_1d_semiconductor c3g_2d_8x8; do
for K in X ACP_QRCP_GRID16; do
env $K=1 timeout 900 python bench.py --config $C --steps 2 --warmup 3 --skip-cpu > gpurun_out/${T}_bench_$C.log 2>&1; echo "bench $C $K rc $? $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/${T}_bench_$C.log | head -1) $(grep -o '"n_mu": [^]]*' gpurun_out/${T}_bench_$C.log | head -1)"
done; done
