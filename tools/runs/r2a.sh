mkdir -p gpurun_out
T=r2a
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc $?"; tail -2 gpurun_out/${T}_pytest.log
timeout 300 python tools/k1_sweep.py c3g_2d_8x8 2048 2>&1 | tail -1
timeout 300 python tools/k1_sweep.py c4g_2d_16x16 2048 2>&1 | tail -1
for C in c3g_2d_8x8 c4g_2d_16x16; do
timeout 1200 python bench.py --config $C --steps 1 --warmup 3 --skip-cpu > gpurun_out/${T}_bench_$C.log 2>&1; echo "bench $C rc $? $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/${T}_bench_$C.log | head -1)"
done
