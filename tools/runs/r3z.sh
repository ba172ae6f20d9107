mkdir -p gpurun_out
T=r3z
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc $?"; tail -1 gpurun_out/${T}_pytest.log
for C in c2_1d_semiconductor c3g_2d_8x8; do
timeout 1800 python bench.py --config $C --steps 2 --warmup 2 --skip-cpu > gpurun_out/${T}_bench_$C.log 2>&1; echo "bench $C rc $? $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/${T}_bench_$C.log | head -1)"
done
