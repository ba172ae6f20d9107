mkdir -p gpurun_out
T=r2o
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "fourier" > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc $?"; tail -1 gpurun_out/${T}_pytest.log
for K in "X=1" "ACP_FFT_GENERIC=1" "X=1" "ACP_FFT_GENERIC=1"; do
echo "$K c1 $(env $K timeout 300 python tools/k1_sweep.py c1_1d_insulator 928 2>&1 | tail -1)"
echo "$K c2 $(env $K timeout 300 python tools/k1_sweep.py c2_1d_semiconductor 2048 2>&1 | tail -1)"
done
for K in "X=1" "ACP_FFT_GENERIC=1"; do
env $K timeout 600 python bench.py --steps 5 --warmup 3 --skip-cpu > gpurun_out/${T}_bench.log 2>&1; echo "bench c1 $K rc $? $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/${T}_bench.log | head -1)"
done
