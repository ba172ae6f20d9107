mkdir -p gpurun_out
T=r2v
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "fourier or tiny2d" > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc $?"; tail -1 gpurun_out/${T}_pytest.log
for r in 1 2; do
echo "c3g $(timeout 300 python tools/k1_sweep.py c3g_2d_8x8 6688 2>&1 | tail -1)"
echo "c4g $(timeout 300 python tools/k1_sweep.py c4g_2d_16x16 4096 2>&1 | tail -1)"
done
timeout 1500 python bench.py --config c3g_2d_8x8 --steps 2 --warmup 3 --skip-cpu > gpurun_out/${T}_bench.log 2>&1; echo "bench c3g rc $? $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/${T}_bench.log | head -1)"
