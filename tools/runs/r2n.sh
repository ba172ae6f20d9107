mkdir -p gpurun_out
T=r2n
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "fourier" > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc $?"; tail -1 gpurun_out/${T}_pytest.log
ACP_FFT_NOKEEP=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "fourier" > gpurun_out/${T}_pytest2.log 2>&1; echo "pytest nokeep rc $?"; tail -1 gpurun_out/${T}_pytest2.log
for K in "X=1" "ACP_FFT_NOKEEP=1" "ACP_FFT_NOKEEP=1 ACP_FFT_THREADS=128" "ACP_FFT_THREADS=192" "ACP_FFT_NOKEEP=1 ACP_FFT_THREADS=256"; do
echo "$K c1 $(env $K timeout 300 python tools/k1_sweep.py c1_1d_insulator 928 2>&1 | tail -1)"
done
for K in "X=1" "ACP_FFT_THREADS=320" "ACP_FFT_THREADS=512" "ACP_FFT_THREADS=1024"; do
echo "$K c2 $(env $K timeout 300 python tools/k1_sweep.py c2_1d_semiconductor 2048 2>&1 | tail -1)"
done
