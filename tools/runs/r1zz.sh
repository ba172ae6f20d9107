mkdir -p gpurun_out
T=r1zz
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "fourier or tiny2d" > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc $?"; tail -2 gpurun_out/${T}_pytest.log
timeout 300 python tools/k1_sweep.py c3g_2d_8x8 2048 2>&1 | tail -1
ACP_FFT2D_CLUSTER=1 timeout 300 python tools/k1_sweep.py c3g_2d_8x8 2048 2>&1 | tail -1
timeout 300 python tools/k1_sweep.py c4g_2d_16x16 2048 2>&1 | tail -1
ACP_FFT2D_CLUSTER=1 timeout 300 python tools/k1_sweep.py c4g_2d_16x16 2048 2>&1 | tail -1
timeout 900 python bench.py --config c3g_2d_8x8 --steps 2 --warmup 3 --skip-cpu > gpurun_out/${T}_bench_c3g.log 2>&1; echo "bench c3g rc $? $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/${T}_bench_c3g.log | head -1)"
