mkdir -p gpurun_out
T=r2k
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc $?"; tail -2 gpurun_out/${T}_pytest.log
for C in c1_1d_insulator c2_1d_semiconductor c3g_2d_8x8; do
for K in X ACP_PCG_GROUPS; do
env $K=1 timeout 1500 python bench.py --config $C --steps 3 --warmup 3 --skip-cpu > gpurun_out/${T}_bench_$C.log 2>&1; echo "bench $C $K rc $? $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/${T}_bench_$C.log | head -1)"
done; done
