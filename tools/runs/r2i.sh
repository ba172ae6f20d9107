mkdir -p gpurun_out
T=r2i
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
for K in "X=1" "ACP_FFT_TWG=1" "ACP_FFT_CARVEOUT=100" "ACP_FFT_TWG=1 ACP_FFT_CARVEOUT=100" "ACP_FFT_TWG=1 ACP_FFT_THREADS=128"; do
echo "$K c1 $(env $K timeout 300 python tools/k1_sweep.py c1_1d_insulator 928 2>&1 | tail -1)"
echo "$K c2 $(env $K timeout 300 python tools/k1_sweep.py c2_1d_semiconductor 2048 2>&1 | tail -1)"
done
