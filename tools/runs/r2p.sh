mkdir -p gpurun_out
T=r2p
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "fourier" > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc $?"; tail -1 gpurun_out/${T}_pytest.log
for K in "X=1" "ACP_FFT_GENERIC=1" "X=1" "ACP_FFT_GENERIC=1"; do
echo "$K c3g $(env $K timeout 300 python tools/k1_sweep.py c3g_2d_8x8 2048 2>&1 | tail -1)"
echo "$K c4g $(env $K timeout 300 python tools/k1_sweep.py c4g_2d_16x16 2048 2>&1 | tail -1)"
done
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/${T}_pytest_all.log 2>&1; echo "pytest all rc $?"; tail -1 gpurun_out/${T}_pytest_all.log
for C in c3g_2d_8x8 c2_1d_semiconductor; do
timeout 1500 python bench.py --config $C --steps 2 --warmup 3 --skip-cpu > gpurun_out/${T}_bench_$C.log 2>&1; echo "bench $C rc $? $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/${T}_bench_$C.log | head -1)"
done
