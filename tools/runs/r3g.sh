mkdir -p gpurun_out
T=r3g
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
ACP_FFT_NOKEEP=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "compiled_lengths" > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc $?"; tail -1 gpurun_out/${T}_pytest.log
for K in X ACP_FFT_NOKEEP X ACP_FFT_NOKEEP; do
echo "$K $(env $K=1 timeout 300 python tools/k1_sweep.py c1_1d_insulator 928 2>&1 | tail -1)"
done
for K in X ACP_FFT_NOKEEP; do
env $K=1 timeout 600 python bench.py --steps 5 --warmup 3 --skip-cpu > gpurun_out/${T}_bench.log 2>&1; echo "c1 $K rc $? $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/${T}_bench.log | head -1)"
done
