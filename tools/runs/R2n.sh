# Round 2, call n: structured Kronecker QRCP: parity (golden, full-m, vs the formed-sketch kernel), timing
mkdir -p gpurun_out
T=${TAG:-R2n}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_golden.py tests/test_gpu_parity.py -q -rs -x -k "golden or full_m or kronecker or large_nmu or compress or dyson_and_dynamical" > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc $?"; tail -15 gpurun_out/${T}_pytest.log
for C in c2_1d_semiconductor c3g_2d_8x8 c4g_2d_16x16; do
for E in X=1 ACP_QRCP_KRON=1 ACP_QRCP_DENSE=1; do
env ${E%%=*}=${E#*=} timeout 300 python tools/qr_time.py $C 2 > gpurun_out/${T}_q.log 2>&1; echo "$E $(tail -1 gpurun_out/${T}_q.log | cut -c1-200)"
done; done
